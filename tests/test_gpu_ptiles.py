"""GPU parity with prefill tiles (F1-F2): K1 fit, K2 prefill
control and K4 simulate on tiled TTFT tables — against the oracle."""
import dataclasses

import numpy as np
import pytest

import synth
from synth.samples import profile_samples
from synth.workload import Layout, Slo

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


def _u32(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to("cuda").view(torch.uint32)


@pytest.mark.parametrize("noise", [0.0, 0.03])
def test_fit_tiled_parity(vt, orc, noise):
    p = synth.make_profile("L8", prefill_tiles=True)
    s = profile_samples(p, 40, 20, noise_sigma=noise, seed=5)
    ref = orc.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], p.k, p.n_tiles,
                          p.tile_w, 0.5, Tp=p.n_ptiles, cutoff=p.prefill_cutoff)
    d = dict(phase=torch.from_numpy(s["phase"]).cuda(),
             level=torch.from_numpy(s["level"].view(np.int16)).cuda().view(torch.uint16),
             n_bt=_u32(s["n_bt"]), n_req=_u32(s["n_req"]), n_kv=_u32(s["n_kv"]),
             lat_ms=torch.from_numpy(s["lat_ms"]).cuda())
    out = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], p.k, p.n_tiles,
                         p.tile_w, 0.5, n_ptiles=p.n_ptiles, prefill_cutoff=p.prefill_cutoff)
    torch.cuda.synchronize()
    assert (out["cell_status"].cpu().numpy() == ref["cell_status"]).all()
    for name in ("a1", "c1", "a2", "b2", "c2", "mae"):
        g, o = out[name].cpu().numpy(), ref[name]
        err = np.abs(g - o) / np.maximum(np.abs(o), 1e-9)
        assert err.max() <= 1e-12 or np.abs(g - o).max() < 1e-12, (name, err.max())


@pytest.mark.parametrize("ladder", [[0, 6, 13, 20, 27], list(range(28)), [13]])
def test_control_step_tiled_prefill(vt, orc, ladder):
    p = synth.make_profile("L8", prefill_tiles=True)
    rng = np.random.default_rng(50 + len(ladder))
    n = 400_000
    load = rng.integers(0, 4000, n).astype(np.uint32)
    load[:1000] = np.repeat([128, 129, 2000, 2001], 250)                 # tile boundaries and the cutoff
    q = np.where(rng.random(n) < 0.1, 1, 0).astype(np.uint32)
    wait = rng.uniform(0, 300, n)
    tgt = rng.uniform(10, 900, n)
    for mode in (0, 1):
        ol, os_ = orc.control_step(p, 0, ladder, load, None, q, wait, tgt, mode=mode)
        lvl, st = vt.control_step(vt.DeviceProfile(p), 0, ladder, _u32(load), None, _u32(q),
                                  torch.from_numpy(wait).cuda(), torch.from_numpy(tgt).cuda(), mode=mode)
        torch.cuda.synchronize()
        assert (st.cpu().numpy() == os_).all()
        assert (lvl.cpu().numpy().astype(np.uint16) == ol).all()


@pytest.mark.parametrize("name,idx,scale", [
    ("C3", list(range(0, 256, 13)), 0.2),
    ("C4", list(range(0, 4096, 197)), 0.15),
])
def test_simulate_tiled_profile(vt, orc, name, idx, scale):
    w = synth.build_config(name, scenarios=idx, duration_scale=scale)
    tiled = [synth.make_profile(p.name if p.name in ("L8", "Q32", "B200", "L8_LINEAR") else "L8", prefill_tiles=True)
             for p in w.profiles]
    w = dataclasses.replace(w, profiles=tiled)
    compare_records(gpu_records(vt, w), orc.simulate_workload(w))


def test_simulate_tiled_and_single_profiles_mixed(vt, orc):
    """Two profiles in one launch, one tiled: the general (non-fast) instantiation."""
    w = synth.build_config("C4", scenarios=list(range(0, 4096, 331)), duration_scale=0.1)
    tiled = synth.make_profile("L8", prefill_tiles=True)
    scen = dict(w.scen, profile_id=(np.arange(w.n) % 2).astype(np.uint32))
    w = dataclasses.replace(w, profiles=[w.profiles[0], tiled], scen=scen)
    compare_records(gpu_records(vt, w), orc.simulate_workload(w))
    p = synth.make_profile("L8", prefill_tiles=True)
    rng = np.random.default_rng(8)
    arr = np.sort(rng.uniform(0, 20000, 300))
    inl = rng.integers(1, 3000, 300)
    outl = rng.integers(1, 200, 300)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(300, 60), Layout(2, 2, max_batch_tokens=2500), [0, 6, 13, 20, 27])
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(300, 60), Layout(1, 1), list(range(28)))
