"""GPU parity for the energy-scored variants (B1-B4):
K2 with mode 1, K3 with policy 2, K4 with policy 2 and/or ctrl_mode 1 — bit-exact
against the oracle like the paper's policies (tests/test_gpu_parity.py)."""
import dataclasses

import numpy as np
import pytest

import synth
from synth.workload import INF_DELTA, Layout, Slo, POLICY_ENERGY, CTRL_ENERGY

from test_gpu_parity import compare_records, gpu_records, _one  # noqa: F401  (fixtures below)

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


@pytest.mark.parametrize("prof_kind,ladder", [("L8", [0, 6, 13, 20, 27]), ("L8", list(range(28))),
                                              ("B200", list(range(60))), ("L8", [13])])
@pytest.mark.parametrize("phase", [0, 1])
def test_control_step_energy_parity(vt, orc, prof_kind, ladder, phase):
    prof = synth.make_profile(prof_kind)
    rng = np.random.default_rng(300 + phase + len(ladder))
    n = 500_000
    load = rng.integers(0, 9000, n).astype(np.uint32)
    load[: n // 4] = rng.integers(1, 16, n // 4)          # light loads: the energy minimum is interior
    kv = (load.astype(np.int64) * rng.integers(0, 900, n)).clip(max=2**32 - 1).astype(np.uint32)
    q = np.where(rng.random(n) < 0.1, rng.integers(1, 50, n), 0).astype(np.uint32)
    wait = rng.uniform(0, 900, n)
    tgt = rng.uniform(1, 900 if phase == 0 else 150, n)
    ol, os_ = orc.control_step(prof, phase, ladder, load, kv, q, wait, tgt, mode=1)
    e0, _ = orc.control_step(prof, phase, ladder, load, kv, q, wait, tgt, mode=0)
    dp = vt.DeviceProfile(prof)
    lvl, st = vt.control_step(dp, phase, ladder, _u32(load), _u32(kv), _u32(q), torch.from_numpy(wait).cuda(),
                              torch.from_numpy(tgt).cuda(), mode=1)
    torch.cuda.synchronize()
    assert (st.cpu().numpy() == os_).all()
    gl = lvl.cpu().numpy().astype(np.uint16)
    assert (gl == ol).all(), np.nonzero(gl != ol)[0][:10]
    if len(ladder) > 1 and phase == 1 and prof_kind == "L8":
        assert (ol != e0).any()                          # the variant is exercised


@pytest.mark.parametrize("n_d", [1, 2, 3, 4, 8])
def test_route_batch_energy_parity(vt, orc, n_d):
    prof = synth.make_profile("L8")
    rng = np.random.default_rng(900 + n_d)
    n = 200_000
    ladder = [0, 6, 13, 20, 27] if n_d != 3 else list(range(28))
    nr = rng.integers(0, 500, (n, n_d)).astype(np.uint32)
    nr[: n // 5] = rng.integers(0, 3, (n // 5, n_d))      # idle / near-idle instances (ties)
    kv = (nr.astype(np.int64) * rng.integers(1, 700, (n, n_d))).astype(np.uint32)
    kv[:50] = 0
    nr[:50, 0] = 5                                        # contract errors (kv < n)
    req_in = rng.integers(1, 4000, n).astype(np.uint32)
    tgt = rng.choice([20.0, 35.0, 45.0, 60.0, 120.0], n)
    cur = rng.integers(0, n_d, n).astype(np.uint32)
    oi, oc, os_, ocur = orc.route_batch(prof, ladder, n_d, nr, kv, req_in, tgt, INF_DELTA, POLICY_ENERGY, cur)
    gcur = _u32(cur.copy())
    gi, gc, gs = vt.route_batch(vt.DeviceProfile(prof), ladder, n_d, _u32(nr), _u32(kv), _u32(req_in),
                                torch.from_numpy(tgt).to("cuda"), INF_DELTA, POLICY_ENERGY, gcur)
    torch.cuda.synchronize()
    assert (gs.cpu().numpy() == os_).all()
    assert (gi.cpu().numpy().astype(np.uint16) == oi).all()
    assert (gc.cpu().numpy() == oc).all()
    assert (gcur.cpu().numpy().astype(np.uint32) == ocur).all()
    if n_d > 1:
        assert {6, 7} <= set(np.unique(oc[os_ == 0]).tolist())


def _energy_variant(w, policy, ctrl, every=1):
    """Layouts i % every == 0 switched to the energy variants (the others stay as built)."""
    lays = [dataclasses.replace(x, policy=policy if (x.policy == 0 and i % every == 0) else x.policy,
                                ctrl_mode=ctrl if i % every == 0 else 0) for i, x in enumerate(w.layouts)]
    return dataclasses.replace(w, layouts=lays)


@pytest.mark.parametrize("policy,ctrl", [(POLICY_ENERGY, 0), (0, CTRL_ENERGY), (POLICY_ENERGY, CTRL_ENERGY)])
@pytest.mark.parametrize("name,idx,scale", [
    ("C3", list(range(0, 256, 11)), 0.2),
    ("C4", list(range(0, 4096, 173)), 0.15),
])
def test_simulate_energy_variants(vt, orc, policy, ctrl, name, idx, scale):
    w = _energy_variant(synth.build_config(name, scenarios=idx, duration_scale=scale), policy, ctrl)
    compare_records(gpu_records(vt, w), orc.simulate_workload(w))


def test_simulate_mixed_default_and_energy(vt, orc):
    """One launch holding default and energy-variant scenarios (the energy instantiation runs
    both); and the default records equal the default-kernel records bit for bit."""
    w0 = synth.build_config("C4", scenarios=list(range(0, 4096, 257)), duration_scale=0.1)
    nl = len(w0.layouts)
    lays = list(w0.layouts) + [dataclasses.replace(x, policy=POLICY_ENERGY, ctrl_mode=CTRL_ENERGY)
                               for x in w0.layouts]
    scen = dict(w0.scen)
    odd = (np.arange(w0.n) % 2) == 1
    scen["layout_id"] = np.where(odd, np.asarray(w0.scen["layout_id"]) + nl, w0.scen["layout_id"]).astype(np.uint32)
    w = dataclasses.replace(w0, layouts=lays, scen=scen)
    g = gpu_records(vt, w)
    compare_records(g, orc.simulate_workload(w))
    g0 = gpu_records(vt, w0)
    assert g[~odd].tobytes() == g0[~odd].tobytes()
    assert g[odd]["decision_hash"].tolist() != g0[odd]["decision_hash"].tolist()


def test_simulate_energy_edge_cases(vt, orc):
    p = synth.make_profile("L8")
    lad5 = [0, 6, 13, 20, 27]
    rng = np.random.default_rng(2)
    arr = np.sort(rng.uniform(0, 20000, 300))
    inl = rng.integers(1, 3000, 300)
    outl = rng.integers(1, 300, 300)
    E = dict(policy=POLICY_ENERGY, ctrl_mode=CTRL_ENERGY)
    _one(vt, orc, np.zeros(0), np.zeros(0), np.zeros(0), 5000.0, p, Slo(600, 60), Layout(2, 2, **E), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 1, **E), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 3, policy=POLICY_ENERGY), list(range(28)))
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60, 0.9), Layout(2, 3, kv_transfer_ms=12.5, **E), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(8, 8, kv_capacity=6000, **E), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(100, 8), Layout(2, 4, **E), lad5)     # mostly infeasible: case 7
    _one(vt, orc, np.repeat(np.arange(30) * 100.0, 10), np.full(300, 128), np.full(300, 129), 4000.0, p,
         Slo(600, 60), Layout(2, 4, **E), lad5)                                        # ties
    b = synth.make_profile("B200")
    _one(vt, orc, arr, inl, outl, 20000.0, b, Slo(100, 10), Layout(4, 4, **E), list(range(60)))
