"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar (BASELINE north_star): decisions, counters and the decision hash bit-exact; fp64
totals within 1e-9 relative (both sides use the same canonical arithmetic, A33, so they
are expected to be bit-exact as well — the count of bit-exact records is asserted too).
Fit coefficients: within 1e-12 relative (fixed-tree vs sequential summation order).
"""

import numpy as np
import pytest

import synth
from synth.profiles import custom_profile
from synth.samples import profile_samples
from synth.workload import INF_DELTA, Layout, Slo, single_trace_workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

INT_FIELDS = ("status", "n_requests", "n_ttft_ok", "n_itl_ok", "n_both_ok", "prefill_iters", "steps_ctrl", "steps_route",
              "decision_hash")
FP_FIELDS = ("sum_ttft_ms", "sum_itl_mean_ms", "e_prefill_busy_j", "e_prefill_idle_j", "e_decode_busy_j",
             "e_decode_idle_j", "busy_ms_prefill", "busy_ms_decode", "top_level_ms", "horizon_ms")


@pytest.fixture(scope="module")
def vt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_04827_b200 as vt
    vt.lib()
    return vt


def compare_records(gpu, orc, rtol=1e-9, require_bitexact=True):
    assert gpu.shape == orc.shape
    for f in INT_FIELDS:
        bad = np.nonzero(gpu[f] != orc[f])[0]
        assert len(bad) == 0, f"{f} differs at {bad[:10]}: gpu {gpu[f][bad[:5]]} oracle {orc[f][bad[:5]]}"
    for f in FP_FIELDS:
        g, o = gpu[f], orc[f]
        err = np.abs(g - o) / np.maximum(np.abs(o), 1e-300)
        assert (err <= rtol).all(), f"{f}: max rel err {err.max()}"
    n_exact = int((gpu.view(np.uint8).reshape(len(gpu), 128) == orc.view(np.uint8).reshape(len(orc), 128))
                  .all(axis=1).sum())
    if require_bitexact:
        assert n_exact == len(gpu), f"only {n_exact}/{len(gpu)} records bit-exact"
    return n_exact


def gpu_records(vt, w):
    return vt.simulate(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)


# ------------------------------------------------------------------ K2 control_step

@pytest.mark.parametrize("prof_kind,ladder", [("L8", [0, 6, 13, 20, 27]), ("L8", list(range(28))),
                                              ("B200", list(range(60))), ("L8", [13]), ("Q32", [0, 27])])
@pytest.mark.parametrize("phase", [0, 1])
def test_control_step_parity(vt, orc, prof_kind, ladder, phase):
    prof = synth.make_profile(prof_kind)
    rng = np.random.default_rng(100 + phase + len(ladder))
    n = 1_000_000
    load = rng.integers(0 if phase == 0 else 0, 9000, n).astype(np.uint32)     # includes contract errors
    kv = (load.astype(np.int64) * rng.integers(0, 900, n)).clip(max=2**32 - 1).astype(np.uint32)
    q = np.where(rng.random(n) < 0.15, rng.integers(1, 50, n), 0).astype(np.uint32)
    wait = rng.uniform(0, 900, n)
    tgt = rng.uniform(1, 900 if phase == 0 else 150, n)
    tgt[:1000] = 60.0                                                            # exact-tie region
    ol, os_ = orc.control_step(prof, phase, ladder, load, kv, q, wait, tgt)
    dp = vt.DeviceProfile(prof)
    T = lambda a, dt: torch.from_numpy(a).to("cuda") if a.dtype != np.uint32 else torch.from_numpy(a.view(np.int32)).to("cuda").view(dt)
    lvl, st = vt.control_step(dp, phase, ladder, T(load, torch.uint32), T(kv, torch.uint32), T(q, torch.uint32),
                              T(wait, None), T(tgt, None))
    torch.cuda.synchronize()
    gl = lvl.cpu().numpy().astype(np.uint16)
    gs = st.cpu().numpy()
    assert (gs == os_).all()
    assert (gl == ol).all(), np.nonzero(gl != ol)[0][:10]


# ------------------------------------------------------------------ K3 route_batch

@pytest.mark.parametrize("n_d", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_route_batch_parity(vt, orc, n_d, policy):
    prof = synth.make_profile("L8")
    rng = np.random.default_rng(7 * n_d + policy)
    n = 200_000
    ladder = [0, 6, 13, 20, 27] if n_d != 3 else list(range(28))
    nr = rng.integers(0, 700, (n, n_d)).astype(np.uint32)
    kv = (nr.astype(np.int64) * rng.integers(1, 700, (n, n_d))).astype(np.uint32)
    kv[:50] = 0                                                                  # contract errors (kv < n)
    req_in = rng.integers(1, 4000, n).astype(np.uint32)
    tgt = rng.choice([40.0, 45.0, 60.0, 80.0, 120.0], n)
    cur = rng.integers(0, n_d, n).astype(np.uint32)
    for delta in (0, 150, 210, INF_DELTA):
        oi, oc, os_, ocur = orc.route_batch(prof, ladder, n_d, nr, kv, req_in, tgt, delta, policy, cur)
        dp = vt.DeviceProfile(prof)
        u32 = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).to("cuda").view(torch.uint32)
        gcur = u32(cur.copy())
        gi, gc, gs = vt.route_batch(dp, ladder, n_d, u32(nr), u32(kv), u32(req_in),
                                    torch.from_numpy(tgt).to("cuda"), delta, policy, gcur)
        torch.cuda.synchronize()
        assert (gs.cpu().numpy() == os_).all()
        assert (gi.cpu().numpy().astype(np.uint16) == oi).all()
        assert (gc.cpu().numpy() == oc).all()
        assert (gcur.cpu().numpy().astype(np.uint32) == ocur).all()


# ------------------------------------------------------------------ K1 fit_profile

@pytest.mark.parametrize("kind,T,noise,n_cell", [("L8", 16, 0.05, 64), ("B200", 4, 0.02, 40), ("Q32", 16, 0.0, 20)])
def test_fit_parity(vt, orc, kind, T, noise, n_cell):
    prof = synth.make_profile(kind, n_tiles=T)
    s = profile_samples(prof, n_cell * 2, n_cell, noise_sigma=noise, seed=11)
    ref = orc.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], prof.k, T, 128, 1.5)
    d = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int32) if v.dtype == np.uint32 else v).to("cuda")
         for k, v in s.items()}
    for k in ("n_bt", "n_req", "n_kv"):
        d[k] = d[k].view(torch.uint32)
    d["level"] = torch.from_numpy(s["level"].view(np.int16)).to("cuda").view(torch.uint16)
    out = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, T, 128, 1.5)
    torch.cuda.synchronize()
    assert (out["cell_status"].cpu().numpy() == ref["cell_status"]).all()
    assert int(out["invalid"].cpu().numpy().view(np.uint64)[0]) == 0
    for name in ("a1", "c1", "a2", "b2", "c2", "mae"):
        g, o = out[name].cpu().numpy(), ref[name]
        err = np.abs(g - o) / np.maximum(np.abs(o), 1e-9)
        assert err.max() <= 1e-12 or np.abs(g - o).max() < 1e-12, (name, err.max())
    # deterministic: a second run is bit-identical
    out2 = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, T, 128, 1.5)
    torch.cuda.synchronize()
    for name in ("a1", "c1", "a2", "b2", "c2", "mae"):
        assert torch.equal(out[name], out2[name])


@pytest.mark.parametrize("kind,T,noise,n_cell", [("L8", 16, 0.05, 96), ("B200", 4, 0.0, 70)])
def test_fit_parity_recording_order(vt, orc, kind, T, noise, n_cell):
    """Samples in recording order (cell by cell, as one profiling run per level records them,
    P:503): most 32-sample chunks are one cell and take K1's lane-tree path; cells of 70 / 96
    samples also leave mixed chunks at every cell boundary."""
    prof = synth.make_profile(kind, n_tiles=T)
    s = profile_samples(prof, n_cell * 2, n_cell, noise_sigma=noise, seed=12, shuffle=False)
    ref = orc.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], prof.k, T, 128, 0.0)
    d = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int32) if v.dtype == np.uint32 else v).to("cuda")
         for k, v in s.items()}
    for k in ("n_bt", "n_req", "n_kv"):
        d[k] = d[k].view(torch.uint32)
    d["level"] = torch.from_numpy(s["level"].view(np.int16)).to("cuda").view(torch.uint16)
    out = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, T, 128, 0.0)
    torch.cuda.synchronize()
    assert (out["cell_status"].cpu().numpy() == ref["cell_status"]).all()
    for name in ("a1", "c1", "a2", "b2", "c2", "mae"):
        g, o = out[name].cpu().numpy(), ref[name]
        err = np.abs(g - o) / np.maximum(np.abs(o), 1e-9)
        assert err.max() <= 1e-12 or np.abs(g - o).max() < 1e-12, (name, err.max())
    out2 = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, T, 128, 0.0)
    torch.cuda.synchronize()
    for name in ("a1", "c1", "a2", "b2", "c2", "mae"):
        assert torch.equal(out[name], out2[name])


def test_fit_degenerate_and_empty(vt, orc):
    prof = synth.make_profile("L8", n_tiles=5)
    s = profile_samples(prof, 10, 12, seed=4, tiles=[0, 1, 2])
    bad = (s["phase"] == 1) & (s["level"] == 5) & (s["n_req"] <= 128)
    s["n_kv"][bad] = 200 * s["n_req"][bad]
    ref = orc.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], prof.k, 5, 128, 2.5)
    u32 = lambda a: torch.from_numpy(a.view(np.int32)).to("cuda").view(torch.uint32)
    out = vt.fit_profile(torch.from_numpy(s["phase"]).cuda(),
                         torch.from_numpy(s["level"].view(np.int16)).cuda().view(torch.uint16),
                         u32(s["n_bt"]), u32(s["n_req"]), u32(s["n_kv"]), torch.from_numpy(s["lat_ms"]).cuda(),
                         prof.k, 5, 128, 2.5)
    assert (out["cell_status"].cpu().numpy() == ref["cell_status"]).all()
    ok = ref["cell_status"] <= 1
    K = prof.k
    for name, sl in (("a2", slice(K, None)), ("c2", slice(K, None))):
        g, o = out[name].cpu().numpy(), ref[name]
        m = ok[sl]
        assert np.allclose(g[m], o[m], rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ K4 simulate

def test_simulate_c1_full(vt, orc):
    w = synth.build_config("C1")
    compare_records(gpu_records(vt, w), orc.simulate_workload(w))


@pytest.mark.parametrize("name,idx,scale", [
    ("C2", list(range(0, 1024, 37)), 0.25),
    ("C3", list(range(0, 256, 9)), 0.2),
    ("C4", list(range(0, 4096, 131)), 0.15),
    ("C5", list(range(0, 16384, 1023)), 0.2),
])
def test_simulate_configs_reduced(vt, orc, name, idx, scale):
    w = synth.build_config(name, scenarios=idx, duration_scale=scale)
    compare_records(gpu_records(vt, w), orc.simulate_workload(w))


@pytest.mark.slow
def test_simulate_c4_full_size_sampled(vt, orc):
    """BASELINE's 4096-scenario sweep at full size (the bench workload, same launch path):
    every GPU record checked by invariants, a stratified sample against the oracle."""
    w = synth.build_config("C4")
    g = gpu_records(vt, w)
    assert (g["status"] == 0).all()
    lens = w.traces.lengths()[w.scen["trace_id"]]
    assert (g["n_requests"] == lens).all()
    assert (g["n_ttft_ok"] <= g["n_requests"]).all() and (g["n_both_ok"] <= g["n_itl_ok"]).all()
    rng = np.random.default_rng(0)
    idx = np.sort(np.concatenate([rng.choice(np.arange(b * 512, (b + 1) * 512), 3, replace=False) for b in range(8)]))
    compare_records(g[idx], orc.simulate_workload(w, idx))


@pytest.mark.slow
@pytest.mark.parametrize("name,n_sample", [("C2", 16), ("C3", 16), ("C5", 12)])
def test_simulate_full_size_sampled(vt, orc, name, n_sample):
    """The other BASELINE configs at full size in one launch each (C5: 16384 scenarios, 4P4D,
    60-level ladder, the general-table instantiation): invariants on every record, a spread
    sample against the oracle."""
    w = synth.build_config(name)
    g = gpu_records(vt, w)
    assert (g["status"] == 0).all()
    assert (g["n_requests"] == w.traces.lengths()[w.scen["trace_id"]]).all()
    assert (g["n_ttft_ok"] <= g["n_requests"]).all() and (g["n_both_ok"] <= g["n_itl_ok"]).all()
    idx = np.unique(np.linspace(0, w.n - 1, n_sample).round().astype(int))
    compare_records(g[idx], orc.simulate_workload(w, idx))


def _one(vt, orc, arrival, inl, outl, D, prof, slo, lay, grid, seed=7):
    w = single_trace_workload(arrival, inl, outl, D, prof, slo, lay, grid, hash_seed=seed)
    g = gpu_records(vt, w)
    o = orc.simulate_workload(w)
    compare_records(g, o)
    return g[0]


def test_simulate_edge_cases(vt, orc):
    p = synth.make_profile("L8")
    lad5 = [0, 6, 13, 20, 27]
    rng = np.random.default_rng(1)
    arr = np.sort(rng.uniform(0, 20000, 300))
    inl = rng.integers(1, 3000, 300)
    outl = rng.integers(1, 300, 300)
    # empty trace
    r = _one(vt, orc, np.zeros(0), np.zeros(0), np.zeros(0), 5000.0, p, Slo(600, 60), Layout(2, 2), lad5)
    assert r["n_requests"] == 0
    # single request; all out == 1; K = 1 static; N_D = 1
    _one(vt, orc, [3.0], [700], [50], 10000.0, p, Slo(600, 60), Layout(1, 1), lad5)
    _one(vt, orc, arr, inl, np.ones(300), 20000.0, p, Slo(600, 60), Layout(2, 2), lad5)
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 2, policy=1), [27])
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(400, 40), Layout(3, 1), list(range(28)))
    # KV transfer delay, Delta = inf, margin s < 1
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60, 0.9), Layout(2, 3, kv_transfer_ms=12.5,
                                                                         delta_mhz=INF_DELTA), lad5)
    # 8P8D (largest template), tiny KV capacity forcing backlog and head-of-line blocking
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(8, 8, kv_capacity=6000), lad5)
    # KV error: a request that can never fit
    r = _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 2, kv_capacity=2500), lad5)
    assert r["status"] == 1
    # tiny batch budget: every batch is a single (oversize) request
    _one(vt, orc, arr, inl, outl, 20000.0, p, Slo(600, 60), Layout(2, 2, max_batch_tokens=1), lad5)
    # simultaneous arrivals and ties
    _one(vt, orc, np.repeat(np.arange(30) * 100.0, 10), np.full(300, 128), np.full(300, 129), 4000.0, p,
         Slo(600, 60), Layout(2, 2), lad5)
    # 60-level ladder (two ballots per evaluation)
    b = synth.make_profile("B200")
    _one(vt, orc, arr, inl, outl, 20000.0, b, Slo(100, 10), Layout(4, 4), list(range(60)))


def test_simulate_wheel_bucket_reuse(vt, orc):
    """Many requests admitted at one START whose finishing iterations alternate between a few
    buckets (out lengths 2,3,2,3,... and long/short mixes), with KV-blocked heads: exercises the
    decode timing wheel's bucket coherence and the cached admission-queue head."""
    p = synth.make_profile("L8")
    n = 600
    arr = np.repeat(np.arange(60) * 50.0, 10)
    outl = np.tile([2, 3, 2, 3, 40, 2, 3, 900, 2, 5], 60)
    outl[7::37] = 1030 + np.arange(len(outl[7::37])) % 3 * 700    # far list: finishes > 1024 ahead
    inl = np.tile([10, 20, 30, 3000, 10, 10, 4000, 10, 10, 20], 60)
    for cap in (400000, 9000):
        _one(vt, orc, arr, inl, outl, 4000.0, p, Slo(600, 60), Layout(1, 2, kv_capacity=cap), [0, 6, 13, 20, 27])
        _one(vt, orc, arr, inl, outl, 4000.0, p, Slo(600, 60), Layout(2, 1, kv_capacity=cap), [0, 27])


def test_simulate_far_list(vt, orc):
    """Many requests finishing more than the wheel's 2048 iterations ahead (out up to 6000): the
    far list's sorted insertion with equal finishing iterations from different admissions, its
    node field holding the finishing iteration, and the in/out restored when a request joins its
    bucket (ITL accounting reads out afterwards), in the default and the variant kernel."""
    p = synth.make_profile("L8")
    rng = np.random.default_rng(11)
    n = 700
    arr = np.sort(rng.uniform(0, 30000, n))
    arr[100:140] = arr[100]                                            # one START admits 40 at once
    outl = rng.integers(1, 200, n)
    outl[::3] = 2050 + rng.integers(0, 3, len(outl[::3])) * 1000      # 2050 / 3050 / 4050: equal fins
    outl[1::29] = 6000
    outl[5::41] = 2050                                                 # exactly at the far threshold
    outl[6::41] = 2049
    inl = rng.integers(1, 2500, n)
    lad5 = [0, 6, 13, 20, 27]
    for lay in (Layout(1, 2), Layout(2, 2, kv_capacity=60000), Layout(3, 1, kv_transfer_ms=3.0),
                Layout(2, 2, itl_mode=2), Layout(1, 3, itl_mode=1, freq_overhead_ms=3.0)):
        _one(vt, orc, arr, inl, outl, 30000.0, p, Slo(600, 60), lay, lad5)


def test_simulate_invalid_trace_status(vt, orc):
    p = synth.make_profile("L8")
    r = _one(vt, orc, [5.0, 1.0], [10, 10], [5, 5], 100.0, p, Slo(600, 60), Layout(1, 1), [0, 27])
    assert r["status"] == 3
    r = _one(vt, orc, [1.0, 5.0], [0, 10], [5, 5], 100.0, p, Slo(600, 60), Layout(1, 1), [0, 27])
    assert r["status"] == 3


def test_simulate_deterministic_and_order_independent(vt, orc):
    w = synth.build_config("C3", scenarios=range(0, 256, 5), duration_scale=0.1)
    a = gpu_records(vt, w)
    wd = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen, order="none")
    wd.launch()
    b = wd.records()
    assert a.tobytes() == b.tobytes()


def test_simulate_prefill_windows_and_completion_log(vt, orc):
    """The split kernel's own paths: K4a's 32-request windows (batches that end inside a window,
    batches re-windowed at their head, batches of more than 32 requests on the general path,
    equal arrival times) and K4b's completion log (many completions per iteration: lists far
    longer than the 4 values a lane gathers; more log chunks than one per lane; an instance that
    gets nearly all the load)."""
    p = synth.make_profile("L8")
    lad5 = [0, 6, 13, 20, 27]
    rng = np.random.default_rng(7)
    # bursts of 1..90 simultaneous short requests: batches of every length around 32 and 64
    sizes = rng.integers(1, 91, 120)
    arr = np.repeat(np.cumsum(rng.uniform(50.0, 400.0, len(sizes))), sizes)
    n = len(arr)
    inl = rng.integers(1, 40, n)
    outl = np.full(n, 60)                     # everything admitted together finishes together
    outl[::17] = rng.integers(2, 400, len(outl[::17]))
    for lay in (Layout(1, 1), Layout(2, 2), Layout(3, 2, max_batch_tokens=300), Layout(1, 2, policy=1)):
        _one(vt, orc, arr, inl, outl, float(arr[-1]) + 1000.0, p, Slo(600, 60), lay, lad5)
    # Delta = 0 with a 2-level ladder: EcoRoute keeps choosing one instance (skewed completion logs)
    _one(vt, orc, arr, inl, outl, float(arr[-1]) + 1000.0, p, Slo(600, 60), Layout(1, 2, delta_mhz=0), [0, 27])


@pytest.mark.parametrize("shuffle", [False, True])
def test_fit_parity_unaligned_and_ragged(vt, orc, shuffle):
    """K1 with sample arrays that start one element into their allocations (no vector loads:
    the element-by-element path) and a count that is not a multiple of the 128-sample chunk."""
    prof = synth.make_profile("L8", n_tiles=6)
    s = profile_samples(prof, 150, 90, noise_sigma=0.03, seed=21, shuffle=shuffle)
    n = len(s["lat_ms"]) - 37
    s = {k: v[:n] for k, v in s.items()}
    ref = orc.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], prof.k, 6, 128, 0.5)

    def dev(a, view=None):
        pad = np.concatenate([a[:1], a])                    # element 0 is padding
        t = torch.from_numpy(pad.view(view) if view else pad).to("cuda")
        return t[1:]

    d = {"phase": dev(s["phase"]), "level": dev(s["level"], np.int16).view(torch.uint16),
         "lat_ms": dev(s["lat_ms"])}
    for k in ("n_bt", "n_req", "n_kv"):
        d[k] = dev(s[k], np.int32).view(torch.uint32)
    out = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, 6, 128, 0.5)
    torch.cuda.synchronize()
    assert (out["cell_status"].cpu().numpy() == ref["cell_status"]).all()
    for name in ("a1", "c1", "a2", "b2", "c2", "mae"):
        g, o = out[name].cpu().numpy(), ref[name]
        err = np.abs(g - o) / np.maximum(np.abs(o), 1e-9)
        assert err.max() <= 1e-12 or np.abs(g - o).max() < 1e-12, (name, err.max())


def test_fit_parity_bench_scale(vt, orc):
    """K1 at the bench's scale: the 2 M-sample calibration set of bench.py (runs of 4201 samples
    per cell, so cell boundaries fall inside 128-sample chunks; a full co-resident grid with its
    barriers) against the oracle's fit of the same samples."""
    import bench
    prof = synth.make_profile("L8")
    s = bench.fit_samples(prof)
    ref = orc.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], prof.k,
                          prof.n_tiles, prof.tile_w, 0.0)
    d = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int32) if v.dtype == np.uint32 else v).to("cuda")
         for k, v in s.items()}
    for k in ("n_bt", "n_req", "n_kv"):
        d[k] = d[k].view(torch.uint32)
    d["level"] = torch.from_numpy(s["level"].view(np.int16)).to("cuda").view(torch.uint16)
    out = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k,
                         prof.n_tiles, prof.tile_w, 0.0)
    torch.cuda.synchronize()
    assert (out["cell_status"].cpu().numpy() == ref["cell_status"]).all()
    for name in ("a1", "c1", "a2", "b2", "c2", "mae"):
        g, o = out[name].cpu().numpy(), ref[name]
        err = np.abs(g - o) / np.maximum(np.abs(o), 1e-9)
        assert err.max() <= 1e-12 or np.abs(g - o).max() < 1e-12, (name, err.max())
