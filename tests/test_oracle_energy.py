"""Pins for the energy-scored variants (readings B1-B4).

PIN-16  energy-argmin controller (ctrl_mode 1): the per-iteration brute force over every
        level sequence of the frequency-control formulation with busy energy
        as the objective, on traces where the load sequence does not depend on the levels.
PIN-17  energy-scored router (policy 2): the north_star's "scores every (candidate
        instance, frequency) successor state ... argmin-energy" enumerated as whole-system
        successor states in exact rational arithmetic, plus the closed-form consolidation
        property of constant power.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import synth
from synth.profiles import custom_profile
from synth.workload import Layout, Slo, INF_DELTA, POLICY_ENERGY, CTRL_ENERGY


def _busy(r):
    return r["e_prefill_busy_j"] + r["e_decode_busy_j"]


# ------------------------------------------------------------------ PIN-16 controller

@pytest.mark.parametrize("prof_name,levels", [("L8", (1005, 1110, 1200, 1410)),
                                               ("B200", None)])
def test_pin16_energy_controller_brute_force(orc, prof_name, levels):
    """One request at a time: the (N_req, N_kv, N_bt) sequence is level-independent, so the
    min-busy-energy feasible level sequence is the per-iteration argmin (separable sum).
    ctrl_mode 1 must reach it exactly; ctrl_mode 0 (EcoFreq) must not when the energy
    minimum is not the lowest feasible level (L8 at N_req = 1)."""
    p = synth.make_profile(prof_name)
    if levels is None:
        lad = np.linspace(0, p.k - 1, 4).round().astype(np.uint16)
    else:
        lad = np.array([p.level_of(f) for f in levels], np.uint16)
    arr, inl, outl = [0.0, 20000.0], [700, 300], [3, 3]
    slo, D = Slo(1e6, 1e6), 40000.0
    lay1 = Layout(1, 1, ctrl_mode=CTRL_ENERGY)
    d1, d0 = {}, {}
    e1 = orc.simulate(np.array(arr), inl, outl, D, slo, lay1, lad, p, diag=d1, iter_cap=64)
    e0 = orc.simulate(np.array(arr), inl, outl, D, slo, Layout(1, 1), lad, p, diag=d0, iter_cap=64)
    n_dec = int(e1["steps_ctrl"])
    assert n_dec == 6
    best = None
    for combo in itertools.product(range(len(lad)), repeat=n_dec):
        dd = {}
        r = orc.simulate(np.array(arr), inl, outl, D, slo, lay1, lad, p, diag=dd, iter_cap=64,
                         force_level=np.array(combo))
        if not (dd["iter_dur"] <= dd["iter_target"]).all():
            continue
        e = _busy(r)
        if best is None or e < best[0]:
            best = (e, combo)
    assert tuple(d1["iter_level"]) == best[1]
    assert abs(_busy(e1) - best[0]) <= 1e-12 * best[0]
    assert _busy(e1) <= _busy(e0) + 1e-12 * _busy(e0)
    if prof_name == "L8":
        assert tuple(d0["iter_level"]) != best[1]         # the variant differs from EcoFreq here


def test_pin16_energy_controller_respects_slo_and_backlog(orc):
    """The SLO mask: every level below the top that the energy controller takes meets its
    target (backlog and nothing-feasible both fall back to the top level, A2/A5)."""
    p = synth.make_profile("L8")
    lad = np.array([p.level_of(f) for f in (1005, 1200, 1410)], np.uint16)
    rng = np.random.default_rng(16)
    arr = np.sort(rng.uniform(0, 3000, 60))
    inl = rng.integers(100, 4000, 60)
    outl = rng.integers(2, 80, 60)
    for slo in (Slo(300.0, 30.0), Slo(2000.0, 60.0), Slo(50.0, 5.0)):
        d = {}
        orc.simulate(arr, inl, outl, 8000.0, slo, Layout(2, 2, ctrl_mode=CTRL_ENERGY), lad, p,
                     diag=d, iter_cap=4096)
        n = len(d["iter_level"])
        lv, dur, tgt = d["iter_level"][:n], d["iter_dur"][:n], d["iter_target"][:n]
        assert n > 0
        # every chosen level below the top met its target
        low = lv < len(lad) - 1
        assert (dur[low] <= tgt[low]).all()


# ------------------------------------------------------------------ PIN-17 router

def _route(orc, p, lad, n, kv, req_in, tgt, cursor=0):
    inst, case, st, cur = orc.route_batch(p, np.asarray(lad, np.uint16), len(n), np.array([n]),
                                          np.array([kv]), [req_in], tgt, INF_DELTA, POLICY_ENERGY,
                                          [cursor])
    assert st[0] == 0
    return int(inst[0]), int(case[0]), int(cur[0])


def _system_brute_force(orc, p, lad, n, kv, req_in, tgt):
    """Enumerate every successor state (d, k): instance d takes the request at level k, every
    other instance keeps EcoFreq's current level (the controller rule, A10/A11). System
    energy rate = sum over instances of P(level, load) * T_itl (0 for an idle instance),
    summed exactly. Mask: the receiving instance's predicted ITL must meet the target."""
    nd, K = len(n), len(lad)

    def rate(level_idx, nn, kk):
        return Fraction(orc.busy_power(p, 1, int(lad[level_idx]), nn)) * \
            Fraction(orc.predict_itl(p, int(lad[level_idx]), nn, kk))

    def ecofreq(nn, kk):
        for k in range(K):
            if orc.predict_itl(p, int(lad[k]), nn, kk) <= tgt:
                return k
        return K - 1

    now = [rate(ecofreq(n[e], kv[e]), n[e], kv[e]) if n[e] > 0 else Fraction(0) for e in range(nd)]
    states = []
    for d in range(nd):
        for k in range(K):
            nn, kk = n[d] + 1, kv[d] + req_in + 1
            if not orc.predict_itl(p, int(lad[k]), nn, kk) <= tgt:
                continue
            total = sum(now[e] for e in range(nd) if e != d) + rate(k, nn, kk)
            states.append((total, d))
    return states


def test_pin17_energy_router_whole_system_brute_force(orc):
    p = synth.make_profile("L8")
    rng = np.random.default_rng(17)
    lad = np.array([0, 6, 13, 20, 27], np.uint16)
    seen_fallback = seen_main = 0
    for it in range(1500):
        nd = int(rng.integers(2, 7))
        n = [int(x) for x in rng.integers(0, 400, nd)]
        kv = [int(x * rng.integers(1, 500)) for x in n]
        req_in = int(rng.integers(1, 3000))
        tgt = float(rng.choice([20.0, 35.0, 45.0, 80.0]))
        cursor = int(rng.integers(nd))
        d, case, cur = _route(orc, p, lad, n, kv, req_in, tgt, cursor)
        states = _system_brute_force(orc, p, lad, n, kv, req_in, tgt)
        if not states:
            # nothing feasible: the fastest top-level successor (B3)
            seen_fallback += 1
            assert case == 7
            tmax = [orc.predict_itl(p, int(lad[-1]), n[e] + 1, kv[e] + req_in + 1) for e in range(nd)]
            assert tmax[d] == min(tmax)
            continue
        seen_main += 1
        assert case == 6
        m = min(s[0] for s in states)
        best_d = {s[1] for s in states if s[0] == m}
        tol = m * Fraction(1, 10**12) if m != 0 else Fraction(1, 10**9)
        near = {s[1] for s in states if s[0] - m <= abs(tol)}
        assert d in near, (n, kv, req_in, tgt, d, best_d)
        if len(near) == 1:
            assert d in best_d
    assert seen_fallback > 20 and seen_main > 500


def test_pin17_energy_router_constant_power_consolidates(orc):
    """Closed form: with constant power P (DYN = 0) and one ITL tile, routing to a busy
    instance adds P*(a2 + b2*(in+1)) while waking an idle one adds P*(a2*1 + b2*(in+1) + c2):
    with c2 > 0 the router packs requests onto already-busy instances until the target
    forces a spill, and identical instances tie (round robin, A17)."""
    K = 2
    p = custom_profile([1005, 1410], np.zeros(K), np.ones(K), np.array([0.1, 0.08]),
                       np.array([1e-4, 1e-4]), np.array([10.0, 8.0]), np.zeros(2 * K),
                       p_idle=100.0, tdp=1e9)
    lad = [0, 1]
    # identical empty instances: a tie -> cursor order, cursor advances
    assert _route(orc, p, lad, [0, 0, 0], [0, 0, 0], 100, 50.0, cursor=1) == (1, 6, 2)
    # one busy instance -> consolidation onto it
    assert _route(orc, p, lad, [0, 5, 0], [0, 900, 0], 100, 50.0, cursor=0)[:2] == (1, 6)
    # the busy instance would violate the target at both levels -> spill to an idle one
    n_full = 400  # 0.08*401 + 1e-4*kv + 8 > 40 at every level
    d, c, _ = _route(orc, p, lad, [n_full, 0], [n_full * 100, 0], 100, 40.0, cursor=0)
    assert (d, c) == (1, 6)
    # two busy instances with different loads: the marginal rate is identical at the same
    # level, so the lower marginal comes from the one that stays at the lower level
    lo = _route(orc, p, lad, [10, 300], [2000, 60000], 100, 38.0, cursor=1)
    assert lo[0] == 0


def test_pin17_single_instance_and_rr_unchanged(orc):
    """policy 2 with N_D = 1 routes to the only instance (A17); policies 0/1 are unaffected."""
    p = synth.make_profile("L8")
    assert _route(orc, p, [0, 27], [5], [500], 10, 40.0)[0] == 0
