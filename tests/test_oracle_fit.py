"""PIN-12: the oracle's EcoPred fitter (least squares per frequency and tile,
PAPER.md:498, :507-518) against closed forms and numpy.linalg.lstsq."""

import numpy as np

import synth
from synth.samples import profile_samples


def _fit(orc, s, prof, tile_step=0.0, T=None):
    return orc.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"],
                           prof.k, T or prof.n_tiles, prof.tile_w, tile_step)


def test_pin12_noiseless_recovery(orc):
    """Noiseless samples from known coefficients are recovered to 1e-9."""
    for kind in ("L8", "Q32"):
        prof = synth.make_profile(kind)
        s = profile_samples(prof, 40, 24, seed=1)
        f = _fit(orc, s, prof)
        assert f["rc"] == 0 and (f["cell_status"] == orc.FIT_OK).all()
        for name in ("a1", "c1", "a2", "b2", "c2"):
            ref = getattr(prof, name)
            assert np.allclose(f[name], ref, rtol=1e-9, atol=0), name
        assert f["mae"].max() < 1e-9


def test_pin12_matches_lstsq(orc):
    """With noise, every cell equals numpy.linalg.lstsq on the same samples (library routine)."""
    prof = synth.make_profile("L8", n_tiles=4)
    s = profile_samples(prof, 50, 30, noise_sigma=0.05, seed=2)
    f = _fit(orc, s, prof)
    assert f["rc"] == 0
    K, T, W = prof.k, prof.n_tiles, prof.tile_w
    for k in range(K):
        m = (s["phase"] == 0) & (s["level"] == k)
        A = np.stack([s["n_bt"][m].astype(float), np.ones(m.sum())], 1)
        coef = np.linalg.lstsq(A, s["lat_ms"][m], rcond=None)[0]
        assert np.allclose([f["a1"][k], f["c1"][k]], coef, rtol=1e-9, atol=1e-11)
        mae = np.abs(s["lat_ms"][m] - A @ coef).mean()
        assert abs(f["mae"][k] - mae) < 1e-9 * mae
        tile = np.minimum(T - 1, (s["n_req"].astype(np.int64) - 1) // W)
        for j in range(T):
            m = (s["phase"] == 1) & (s["level"] == k) & (tile == j)
            A = np.stack([s["n_req"][m].astype(float), s["n_kv"][m].astype(float), np.ones(m.sum())], 1)
            coef = np.linalg.lstsq(A, s["lat_ms"][m], rcond=None)[0]
            o = j * K + k
            got = np.array([f["a2"][o], f["b2"][o], f["c2"][o]])
            assert np.allclose(got, coef, rtol=1e-8, atol=1e-10), (k, j, got, coef)


def test_pin12_collinear_cell_is_degenerate(orc):
    """n_kv = 200 n_req everywhere in a cell -> calibration error naming the cell."""
    prof = synth.make_profile("L8", n_tiles=2)
    s = profile_samples(prof, 10, 10, seed=3)
    bad = (s["phase"] == 1) & (s["level"] == 5) & (s["n_req"] <= 128)
    s["n_kv"][bad] = 200 * s["n_req"][bad]
    f = _fit(orc, s, prof)
    assert f["rc"] == 4
    st = f["cell_status"]
    assert st[prof.k + 0 * prof.k + 5] == orc.FIT_DEGENERATE
    assert (np.delete(st, prof.k + 5) == orc.FIT_OK).all()


def test_pin12_empty_cells(orc):
    """Empty ITL tiles inherit the lower tile + step; an empty TTFT level or tile 0
    is an error naming it."""
    prof = synth.make_profile("L8", n_tiles=5)
    s = profile_samples(prof, 10, 12, seed=4, tiles=[0, 1, 2])
    f = _fit(orc, s, prof, tile_step=2.5)
    K = prof.k
    assert f["rc"] == 0
    for j in (3, 4):
        for k in range(K):
            o, pv = j * K + k, (j - 1) * K + k
            assert f["cell_status"][K + o] == orc.FIT_INHERITED
            assert f["a2"][o] == f["a2"][pv] and f["b2"][o] == f["b2"][pv]
            assert f["c2"][o] == f["c2"][pv] + 2.5
    s = profile_samples(prof, 10, 12, seed=5, levels=[0, 1, 3])
    f = orc.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], 4, 5, 128, 0.0)
    assert f["rc"] == 4 and f["cell_status"][2] == orc.FIT_EMPTY and f["cell_status"][4 + 2] == orc.FIT_EMPTY


def test_pin12_noisy_mae_bound(orc):
    """Multiplicative noise sigma = 0.05: held-out MAE below 3x the noise floor,
    the paper's single-digit-ms regime."""
    prof = synth.make_profile("L8", n_tiles=4)
    sig = 0.05
    tr = profile_samples(prof, 200, 120, noise_sigma=sig, seed=6)
    f = _fit(orc, tr, prof)
    te = profile_samples(prof, 200, 120, noise_sigma=sig, seed=7)
    clean = profile_samples(prof, 200, 120, noise_sigma=0.0, seed=7)
    K, T, W = prof.k, prof.n_tiles, prof.tile_w
    ph, lv = te["phase"], te["level"].astype(int)
    tile = np.minimum(T - 1, (te["n_req"].astype(np.int64) - 1) // W)
    o = np.where(ph == 1, tile * K + lv, 0)
    yh = np.where(ph == 0, f["a1"][lv] * te["n_bt"] + f["c1"][lv],
                  f["a2"][o] * te["n_req"] + f["b2"][o] * te["n_kv"] + f["c2"][o])
    for p_ in (0, 1):
        m = ph == p_
        mae = np.abs(te["lat_ms"][m] - yh[m]).mean()
        floor = np.abs(te["lat_ms"][m] - clean["lat_ms"][m]).mean()
        assert mae < 3 * floor, (p_, mae, floor)
