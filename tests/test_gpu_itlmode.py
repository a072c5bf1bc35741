"""GPU parity of the ITL Max / nearest-rank P99 attainment modes (E3; PIN-23),
alone and with the other variants, against the oracle (which sorts every request's gaps)."""
import dataclasses

import numpy as np
import pytest

import synth
from synth.workload import Layout, Slo, POLICY_ENERGY

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


@pytest.mark.parametrize("kw", [
    dict(itl_mode=1), dict(itl_mode=2),
    dict(itl_mode=1, freq_overhead_ms=50.0), dict(itl_mode=2, freq_overhead_ms=3.0, ctrl_interval_ms=300.0),
    dict(itl_mode=2, policy=POLICY_ENERGY, exec_noise=synth.exec_noise_table(0.1, 1024)),
])
@pytest.mark.parametrize("name,idx,scale", [
    ("C3", list(range(0, 256, 23)), 0.2),
    ("C4", list(range(0, 4096, 257)), 0.15),
])
def test_simulate_itl_modes(vt, orc, kw, name, idx, scale):
    w = synth.build_config(name, scenarios=idx, duration_scale=scale)
    w = dataclasses.replace(w, layouts=[dataclasses.replace(x, **kw) for x in w.layouts])
    g = gpu_records(vt, w)
    o = orc.simulate_workload(w)
    compare_records(g, o)


def test_itl_modes_edge_cases(vt, orc):
    p = synth.make_profile("L8")
    lad5 = [0, 6, 13, 20, 27]
    rng = np.random.default_rng(5)
    arr = np.sort(rng.uniform(0, 20000, 300))
    inl = rng.integers(1, 3000, 300)
    outl = rng.integers(1, 300, 300)
    for m in (1, 2):
        _one(vt, orc, [0.0], [100], [102], 0.0, p, Slo(1e6, 25.0), Layout(1, 1, freq_overhead_ms=50.0, itl_mode=m),
             lad5)
        _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 30), Layout(2, 2, itl_mode=m, kv_transfer_ms=7.5), lad5)
        _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 30), Layout(8, 8, kv_capacity=6000, itl_mode=m), lad5)
        long_out = np.where(np.arange(300) % 17 == 0, 1500, outl)          # windows past the wheel (far list)
        _one(vt, orc, arr, inl, long_out, 20000.0, p, Slo(600, 30), Layout(1, 2, itl_mode=m), lad5)
