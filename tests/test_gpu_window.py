"""GPU parity for window-interval control and blocking frequency-set overhead (SURVEY.md §8(f)
row f2; C1-C4), alone and combined with the energy variants — bit-exact against
the oracle."""
import dataclasses

import numpy as np
import pytest

import synth
from synth.workload import Layout, Slo, POLICY_ENERGY, CTRL_ENERGY

from test_gpu_parity import compare_records, gpu_records, _one  # noqa: F401

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_04827_b200 as vt
    vt.lib()
    return vt


def _variant(w, **kw):
    return dataclasses.replace(w, layouts=[dataclasses.replace(x, **kw) for x in w.layouts])


@pytest.mark.parametrize("kw", [
    dict(ctrl_interval_ms=1000.0),
    dict(ctrl_interval_ms=5000.0),
    dict(freq_overhead_ms=3.0),
    dict(freq_overhead_ms=50.0),
    dict(ctrl_interval_ms=250.0, freq_overhead_ms=50.0),
    dict(ctrl_interval_ms=1000.0, freq_overhead_ms=3.0, policy=POLICY_ENERGY, ctrl_mode=CTRL_ENERGY),
])
@pytest.mark.parametrize("name,idx,scale", [
    ("C3", list(range(0, 256, 13)), 0.2),
    ("C4", list(range(0, 4096, 211)), 0.15),
])
def test_simulate_window_overhead_variants(vt, orc, kw, name, idx, scale):
    w = _variant(synth.build_config(name, scenarios=idx, duration_scale=scale), **kw)
    g = gpu_records(vt, w)
    o = orc.simulate_workload(w)
    compare_records(g, o)


def test_simulate_window_edge_cases(vt, orc):
    p = synth.make_profile("L8")
    lad5 = [0, 6, 13, 20, 27]
    rng = np.random.default_rng(3)
    arr = np.sort(rng.uniform(0, 20000, 300))
    inl = rng.integers(1, 3000, 300)
    outl = rng.integers(1, 300, 300)
    _one(vt, orc, np.zeros(0), np.zeros(0), np.zeros(0), 5000.0, p, Slo(600, 60),
         Layout(2, 2, ctrl_interval_ms=100.0, freq_overhead_ms=50.0), lad5)
    _one(vt, orc, [3.0], [700], [50], 10000.0, p, Slo(600, 60), Layout(1, 1, freq_overhead_ms=50.0), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 2, ctrl_interval_ms=1e11), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 2, freq_overhead_ms=50.0), [27])   # K = 1
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60, 0.9),
         Layout(2, 3, kv_transfer_ms=12.5, freq_overhead_ms=3.0, ctrl_interval_ms=40.0), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60),
         Layout(8, 8, kv_capacity=6000, freq_overhead_ms=50.0, ctrl_interval_ms=500.0), lad5)
    r = _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 2, kv_capacity=2500, freq_overhead_ms=5.0),
             lad5)
    assert r["status"] == 1
    _one(vt, orc, np.repeat(np.arange(30) * 100.0, 10), np.full(300, 128), np.full(300, 129), 4000.0, p,
         Slo(600, 60), Layout(2, 2, ctrl_interval_ms=100.0, freq_overhead_ms=3.0), lad5)   # ties on the boundary
    b = synth.make_profile("B200")
    _one(vt, orc, arr, inl, outl, 20000.0, b, Slo(100, 10),
         Layout(4, 4, ctrl_interval_ms=300.0, freq_overhead_ms=3.0, policy=POLICY_ENERGY), list(range(60)))
