"""PIN-21: the fit -> simulate loop (E4).

Simulated iterations are calibration samples (P:498 offline profiling, here of the simulated
system). S:170 "fit∘generate is the identity on noiseless synthetic data": fitting the
oracle's noiseless iteration log recovers the generating profile's coefficients on every
fitted cell; with multiplicative lognormal noise of log-sd sigma the per-cell MAE is about
E|eps - 1| * latency = sigma * sqrt(2/pi) * latency.
"""
import dataclasses

import numpy as np

import synth


def log_samples(d, ladder, n_p):
    """Oracle iteration log -> EcoPred sample SoA (the mapping voltana_series_to_samples states)."""
    inst = d["iter_inst"]
    phase = (inst >= n_p).astype(np.uint8)
    level = np.asarray(ladder, np.uint16)[d["iter_level"]]
    n_bt = np.where(phase == 0, d["iter_load"], 0).astype(np.uint32)
    n_req = np.where(phase == 1, d["iter_load"], 0).astype(np.uint32)
    n_kv = np.where(phase == 1, d["iter_kv"], 0).astype(np.uint32)
    return phase, level, n_bt, n_req, n_kv, d["iter_dur"].copy()


def _run(orc, w, sigma):
    out = []
    for c in range(w.n):
        s = w.scen
        a, ii, o, D = w.traces.trace(int(s["trace_id"][c]))
        lay = w.layouts[s["layout_id"][c]]
        if sigma > 0:
            lay = dataclasses.replace(lay, exec_noise=synth.exec_noise_table(sigma, 4096, seed=c))
        d = {}
        r = orc.simulate(a, ii, o, D, w.slos[s["slo_id"][c]], lay, w.grids[s["grid_id"][c]], w.profiles[0],
                         int(s["hash_seed"][c]), diag=d, iter_cap=1 << 22)
        assert r["status"] == 0
        out.append(log_samples(d, w.grids[s["grid_id"][c]], lay.n_p))
    return [np.concatenate([o[i] for o in out]) for i in range(6)]


def test_pin21_noiseless_loop_recovers_profile(orc):
    w = synth.build_config("C4", scenarios=list(range(3584, 4096, 64)), duration_scale=0.3)   # high rates
    p = w.profiles[0]
    smp = _run(orc, w, 0.0)
    f = orc.fit_profile(*smp, p.k, p.n_tiles, p.tile_w, 0.0)
    K = p.k
    st = f["cell_status"]
    ok_t = np.nonzero(st[:K] == 0)[0]
    ok_i = np.nonzero(st[K:] == 0)[0]
    assert len(ok_t) >= 3 and len(ok_i) >= 4
    for name, ref, idx in (("a1", p.a1, ok_t), ("c1", p.c1, ok_t), ("a2", p.a2, ok_i), ("b2", p.b2, ok_i),
                           ("c2", p.c2, ok_i)):
        err = np.abs(f[name][idx] - ref[idx]) / np.abs(ref[idx])
        assert err.max() < 1e-9, (name, err.max())
    assert f["mae"][np.concatenate([ok_t, K + ok_i])].max() < 1e-9


def test_pin21_noisy_loop_mae_matches_noise_floor(orc):
    sigma = 0.05
    w = synth.build_config("C4", scenarios=list(range(3584, 4096, 64)), duration_scale=0.3)
    p = w.profiles[0]
    phase, level, n_bt, n_req, n_kv, lat = _run(orc, w, sigma)
    f = orc.fit_profile(phase, level, n_bt, n_req, n_kv, lat, p.k, p.n_tiles, p.tile_w, 0.0)
    K = p.k
    floor = sigma * np.sqrt(2 / np.pi)
    checked = 0
    for c in range(K + p.n_tiles * K):
        if f["cell_status"][c] != 0:
            continue
        if c < K:
            m = (phase == 0) & (level == c)
        else:
            j, lv = divmod(c - K, K)
            m = (phase == 1) & (level == lv) & (np.minimum((n_req.astype(np.int64) - 1) // p.tile_w, p.n_tiles - 1) == j)
        if m.sum() < 200:
            continue
        rel = f["mae"][c] / lat[m].mean()
        assert 0.6 * floor < rel < 1.5 * floor, (c, rel, floor)
        checked += 1
    assert checked >= 3
