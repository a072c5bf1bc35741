"""GPU parity with execution noise (D1-D3), alone and with
the other variants — bit-exact against the oracle (the factors come from the same input
table through the same counter-based index)."""
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


@pytest.mark.parametrize("sigma,n,extra", [
    (0.05, 4096, {}),
    (0.3, 1024, {}),
    (0.1, 1, {}),
    (0.05, 4096, dict(ctrl_interval_ms=500.0, freq_overhead_ms=3.0)),
    (0.05, 4096, dict(policy=POLICY_ENERGY, ctrl_mode=CTRL_ENERGY)),
])
@pytest.mark.parametrize("name,idx,scale", [
    ("C3", list(range(0, 256, 17)), 0.2),
    ("C4", list(range(0, 4096, 239)), 0.15),
])
def test_simulate_noise_parity(vt, orc, sigma, n, extra, name, idx, scale):
    w = synth.build_config(name, scenarios=idx, duration_scale=scale)
    tab = synth.exec_noise_table(sigma, n=n, seed=1)
    w = dataclasses.replace(w, layouts=[dataclasses.replace(x, exec_noise=tab, **extra) for x in w.layouts])
    g = gpu_records(vt, w)
    o = orc.simulate_workload(w)
    compare_records(g, o)


def test_simulate_noise_edge_cases(vt, orc):
    p = synth.make_profile("L8")
    lad5 = [0, 6, 13, 20, 27]
    rng = np.random.default_rng(4)
    arr = np.sort(rng.uniform(0, 20000, 300))
    inl = rng.integers(1, 3000, 300)
    outl = rng.integers(1, 300, 300)
    tab = synth.exec_noise_table(0.2, n=256, seed=2)
    _one(vt, orc, np.zeros(0), np.zeros(0), np.zeros(0), 5000.0, p, Slo(600, 60), Layout(2, 2, exec_noise=tab), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(8, 8, kv_capacity=6000, exec_noise=tab), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 3, kv_transfer_ms=12.5, exec_noise=tab), lad5)
    bad = tab.copy()
    bad[::7] = 0.0
    r = _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 2, exec_noise=bad), lad5)
    assert r["status"] == 3
    r = _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 2, exec_noise=np.full(4, np.nan)), lad5)
    assert r["status"] == 3
