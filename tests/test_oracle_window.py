"""Pins for window-interval control and blocking frequency-set overhead (
DESIGN.md readings C1-C4).

PIN-18  gating: decisions happen exactly when the elapsed time since the previous decision
        reaches the interval (inclusive, S:281-289 examples), counted on traces with exact
        binary times; a reconstruction of the gating rule from the iteration log; levels only
        change at decisions.
PIN-19  blocking overhead: closed-form single-request trace; the overhead
        is paid only on a level change; iteration-log timing invariants.
"""
import numpy as np
import pytest

import synth
from synth.profiles import custom_profile
from synth.workload import Layout, Slo


def _flat2(c1=(100.0, 60.0), c2=(20.0, 12.0)):
    """Two levels, constant predictions (a = b = 0): TT = c1[k], IT = c2[k]."""
    K = 2
    z = np.zeros(K)
    return custom_profile([1005, 1410], z, np.array(c1, float), z, z, np.array(c2, float),
                          np.array([100.0, 200.0, 50.0, 90.0]), p_idle=60.0, tdp=1e9)


def _sim(orc, prof, arr, inl, outl, D, slo, lay, lad=(0, 1), **kw):
    return orc.simulate(np.asarray(arr, float), np.asarray(inl), np.asarray(outl), D, slo, lay,
                        np.asarray(lad, np.uint16), prof, **kw)


# ------------------------------------------------------------------ PIN-18 gating

@pytest.mark.parametrize("interval,it_ms,n_iter,expect_dec", [
    (0.0, 10.0, 12, 12),          # per-iteration ("interval 0 -> decision every call")
    (30.0, 10.0, 12, 4),          # starts 0,10,..,110: decisions at 0,30,60,90 (boundary inclusive)
    (30.5, 10.0, 12, 3),          # decisions at 0,40,80
    (1e9, 10.0, 12, 1),           # one decision for the whole run
    (5000.0, 1250.0, 6, 2),       # elapsed 1250..3750 -> no change; elapsed 5000 -> fresh
])
def test_pin18_window_decision_count(orc, interval, it_ms, n_iter, expect_dec):
    prof = _flat2(c1=(100.0, 60.0), c2=(it_ms, it_ms / 2))
    r = _sim(orc, prof, [0.0], [100], [n_iter + 1], 0.0, Slo(1e6, 1e6),
             Layout(1, 1, ctrl_interval_ms=interval))
    assert r["status"] == 0
    assert r["steps_route"] == 1
    assert r["steps_ctrl"] == 1 + expect_dec            # + the one prefill decision
    assert r["prefill_iters"] == 1


def _reconstruct_decisions(log, interval):
    """Gating rule restated on the iteration log: per instance, the first iteration decides,
    then every iteration whose START is >= interval after the previous deciding START."""
    dec = np.zeros(len(log["iter_inst"]), bool)
    last = {}
    for i, (inst, t) in enumerate(zip(log["iter_inst"], log["iter_start"])):
        if inst not in last or t - last[inst] >= interval:
            dec[i] = True
            last[inst] = t
    return dec


@pytest.mark.parametrize("interval", [0.0, 25.0, 200.0, 1000.0, 5000.0])
def test_pin18_window_gating_reconstructed(orc, interval):
    p = synth.make_profile("L8")
    rng = np.random.default_rng(18)
    m = 250
    arr = np.sort(rng.uniform(0, 15000, m))
    inl = rng.integers(20, 3000, m)
    outl = rng.integers(1, 120, m)
    lad = np.array([0, 6, 13, 20, 27], np.uint16)
    d = {}
    r = orc.simulate(arr, inl, outl, 15000.0, Slo(400.0, 40.0), Layout(2, 2, ctrl_interval_ms=interval), lad, p,
                     diag=d, iter_cap=200000)
    assert r["status"] == 0
    n = len(d["iter_inst"])
    assert n == int(r["prefill_iters"]) + int(d["iters"][2:].sum())
    dec = _reconstruct_decisions(d, interval)
    assert int(dec.sum()) == int(r["steps_ctrl"])
    # levels change only at decisions (a carried level is the previous iteration's level)
    prev = {}
    for i in range(n):
        inst, lv = int(d["iter_inst"][i]), int(d["iter_level"][i])
        if not dec[i]:
            assert lv == prev[inst]
        prev[inst] = lv
    if interval == 0.0:
        assert dec.all()
    if interval >= 1000.0:
        assert (~dec).sum() > n // 2


def test_pin18_window_zero_is_per_iteration(orc):
    """interval 0 and overhead 0 reproduce the per-iteration controller bit for bit."""
    for w in (synth.build_config("C1"), synth.build_config("C3", scenarios=range(0, 256, 51), duration_scale=0.2)):
        for i in range(w.n):
            a, ii, o, D = w.traces.trace(int(w.scen["trace_id"][i]))
            lay = w.layouts[w.scen["layout_id"][i]]
            args = (a, ii, o, D, w.slos[w.scen["slo_id"][i]])
            base = orc.simulate(*args, lay, w.grids[w.scen["grid_id"][i]], w.profiles[0], 5)
            import dataclasses
            lay0 = dataclasses.replace(lay, ctrl_interval_ms=0.0, freq_overhead_ms=0.0)
            again = orc.simulate(*args, lay0, w.grids[w.scen["grid_id"][i]], w.profiles[0], 5)
            assert base.tobytes() == again.tobytes()


# ------------------------------------------------------------------ PIN-19 blocking overhead

def test_pin19_overhead_single_request_closed_form(orc):
    """Loose SLO: EcoFreq picks level 0 everywhere; the GPU starts at the top level (C2), so
    each instance pays the overhead once, at its first iteration:
      TTFT = ov + c1[0];  t_done = TTFT + ov + (out-1)*c2[0];  ITL mean = (ov + (out-1) c2[0]) / (out-1).
    Busy time and busy energy are those of the overhead-free run."""
    prof = _flat2()
    out, ov = 5, 50.0
    base = _sim(orc, prof, [0.0], [100], [out], 0.0, Slo(1e6, 1e6), Layout(1, 1))
    d = {}
    r = _sim(orc, prof, [0.0], [100], [out], 0.0, Slo(1e6, 1e6), Layout(1, 1, freq_overhead_ms=ov),
             diag=d)
    assert d["req_tfirst"][0] == ov + 100.0 == 150.0
    assert d["req_tdone"][0] == 150.0 + ov + (out - 1) * 20.0 == 280.0
    assert d["req_itl"][0] == (ov + (out - 1) * 20.0) / (out - 1) == 32.5
    assert r["sum_ttft_ms"] == 150.0 and r["horizon_ms"] == 280.0
    for f in ("busy_ms_prefill", "busy_ms_decode", "e_prefill_busy_j", "e_decode_busy_j", "steps_ctrl",
              "decision_hash"):
        assert r[f] == base[f], f
    # idle energy grows by p_idle * (extra horizon) per instance (A24 idle = horizon - busy)
    extra = (280.0 - 180.0)
    assert abs((r["e_prefill_idle_j"] + r["e_decode_idle_j"]) - (base["e_prefill_idle_j"] + base["e_decode_idle_j"])
               - 2 * 60.0 * extra / 1000.0) < 1e-12


def test_pin19_no_overhead_without_level_change(orc):
    """Tight SLO keeps every decision at the top level = the starting level: no overhead at all
    (S:452 'unchanged frequency -> zero overhead in both modes')."""
    prof = _flat2()
    slo = Slo(80.0, 15.0)                    # level 0 (100 ms / 20 ms) infeasible, level 1 feasible
    base = _sim(orc, prof, [0.0, 500.0], [100, 100], [6, 6], 0.0, slo, Layout(1, 1))
    r = _sim(orc, prof, [0.0, 500.0], [100, 100], [6, 6], 0.0, slo, Layout(1, 1, freq_overhead_ms=50.0))
    assert r.tobytes() == base.tobytes()


@pytest.mark.parametrize("ov,interval", [(3.0, 0.0), (50.0, 0.0), (50.0, 500.0)])
def test_pin19_overhead_log_invariants(orc, ov, interval):
    p = synth.make_profile("L8")
    rng = np.random.default_rng(19)
    m = 200
    arr = np.sort(rng.uniform(0, 12000, m))
    inl = rng.integers(20, 3000, m)
    outl = rng.integers(1, 100, m)
    lad = np.array([0, 6, 13, 20, 27], np.uint16)
    d = {}
    r = orc.simulate(arr, inl, outl, 12000.0, Slo(500.0, 45.0),
                     Layout(2, 2, freq_overhead_ms=ov, ctrl_interval_ms=interval), lad, p, diag=d, iter_cap=200000)
    assert r["status"] == 0
    K = len(lad)
    cur, free = {}, {}
    n_paid = 0
    for inst, lv, t, dur in zip(d["iter_inst"], d["iter_level"], d["iter_start"], d["iter_dur"]):
        inst, lv = int(inst), int(lv)
        assert t >= free.get(inst, -1.0)                 # an instance starts only when free
        paid = lv != cur.get(inst, K - 1)
        n_paid += paid
        free[inst] = (t + ov if paid else t) + dur
        cur[inst] = lv
    assert n_paid > 0
    assert r["horizon_ms"] >= max(free.values())
    assert r["busy_ms_prefill"] + r["busy_ms_decode"] == pytest.approx(float(d["iter_dur"].sum()), rel=1e-12)


def test_pin19_paper_ablation_direction(orc):
    """Behaviour: on a bursty 1P1D ShareGPT-like trace, 5-s window control
    lowers TTFT attainment relative to per-iteration control, and a blocking 50-ms frequency
    set lowers attainment relative to a 3-ms one."""
    p = synth.make_profile("L8")
    w = synth.build_config("C3", scenarios=[5], duration_scale=0.5)
    a, ii, o, D = w.traces.trace(int(w.scen["trace_id"][0]))
    lad = np.array([0, 6, 13, 20, 27], np.uint16)
    slo = Slo(600.0, 45.0)
    per_it = orc.simulate(a, ii, o, D, slo, Layout(1, 1), lad, p)
    win = orc.simulate(a, ii, o, D, slo, Layout(1, 1, ctrl_interval_ms=5000.0), lad, p)
    fast = orc.simulate(a, ii, o, D, slo, Layout(1, 1, freq_overhead_ms=3.0), lad, p)
    slow = orc.simulate(a, ii, o, D, slo, Layout(1, 1, freq_overhead_ms=50.0), lad, p)
    assert win["n_ttft_ok"] < per_it["n_ttft_ok"]
    assert slow["n_both_ok"] < fast["n_both_ok"]
