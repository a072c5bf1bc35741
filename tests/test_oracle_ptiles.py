"""PIN-22: prefill tiles (Appendix B; SPEC.md:99-100,
S:174; readings F1-F2).

"We can observe similar staircase-like boundary effect like decode phase ... this effect only
exist when number of batched tokens are relative small. When number of batched tokens goes
over about 2000, this effect gradually becomes less significant." The TTFT model gets one
coefficient pair per prefill tile below the cutoff and one linear tile above it.
"""
import numpy as np
import pytest

import synth
from synth.profiles import custom_profile
from synth.samples import profile_samples
from synth.workload import Layout, Slo


def _tiled(tp=17, cutoff=2000):
    p = synth.make_profile("L8", prefill_tiles=True)
    assert p.n_ptiles == tp and p.prefill_cutoff == cutoff
    return p


def test_pin22_prefill_tile_index_examples(orc):
    p = _tiled()
    # W = 128, cutoff 2000, T_p = ceil(2000/128) + 1 = 17: tiles 0..15 below the cutoff, 16 above
    for nbt, j in ((1, 0), (128, 0), (129, 1), (256, 1), (257, 2), (1920, 14), (1921, 15), (2000, 15),
                   (2001, 16), (8192, 16), (10 ** 6, 16)):
        assert orc.ptile_index(p, nbt) == j, nbt
    single = synth.make_profile("L8")
    assert single.n_ptiles == 1
    assert all(orc.ptile_index(single, x) == 0 for x in (1, 129, 2001, 9000))


def test_pin22_prediction_uses_the_tile_row(orc):
    """Hand-built tiled tables: TTFT(k, nbt) = a1[jp][k]*nbt + c1[jp][k] exactly (eq:pred-ttft,
    P:514), with the staircase jump at the 128 -> 129 boundary and the linear tile above 2000."""
    K, tp = 2, 17
    a1 = np.tile([0.25, 0.125], tp)
    c1 = np.concatenate([[8.0 + jp, 4.0 + jp] for jp in range(tp)])
    p = custom_profile([1005, 1410], a1, c1, np.zeros(K), np.zeros(K), np.ones(K), np.full(2 * K, 100.0))
    p.n_ptiles, p.prefill_cutoff = tp, 2000
    assert orc.predict_ttft(p, 0, 128) == 0.25 * 128 + 8.0 == 40.0
    assert orc.predict_ttft(p, 0, 129) == 0.25 * 129 + 9.0 == 41.25        # one tile up: +a1 +1 ms step
    assert orc.predict_ttft(p, 1, 2000) == 0.125 * 2000 + 19.0 == 269.0     # tile 15
    assert orc.predict_ttft(p, 1, 2001) == 0.125 * 2001 + 20.0              # the large tile 16
    # a single request's TTFT in the simulation is the tile-row prediction
    r = orc.simulate(np.array([0.0]), [129], [1], 0.0, Slo(1e6, 1e6), Layout(1, 1), np.array([0], np.uint16), p)
    assert r["sum_ttft_ms"] == 41.25


def test_pin22_staircase_profile_is_monotone(orc):
    """The synthetic tiled profile steps up at each boundary below the cutoff (Appendix B) and is
    continuous-from-below linear above it; at fixed N_bt, higher levels are never slower."""
    p = _tiled()
    for k in (0, 13, 27):
        prev = None
        for nbt in range(1, 2600, 7):
            t = orc.predict_ttft(p, k, nbt)
            if prev is not None:
                assert t >= prev
            prev = t
        assert orc.predict_ttft(p, k, 129) - orc.predict_ttft(p, k, 128) > p.a1[k]   # the step
    for nbt in (50, 700, 1999, 2001, 5000):
        t = [orc.predict_ttft(p, k, nbt) for k in range(p.k)]
        assert all(a >= b for a, b in zip(t, t[1:]))


def test_pin22_fit_recovers_tiled_profile(orc):
    """Noiseless samples of a tiled profile: every (prefill tile, level) cell is recovered to
    1e-9 (S:153 exact recovery); an empty prefill tile inherits the previous one + step (F2)."""
    p = _tiled()
    s = profile_samples(p, 12, 8, seed=22)
    f = orc.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], p.k, p.n_tiles,
                        p.tile_w, 0.0, Tp=p.n_ptiles, cutoff=p.prefill_cutoff)
    assert f["rc"] == 0
    kp = p.n_ptiles * p.k
    assert (f["cell_status"][:kp] == 0).all()
    for name in ("a1", "c1"):
        err = np.abs(f[name] - getattr(p, name)) / np.abs(getattr(p, name))
        assert err.max() < 1e-9, (name, err.max())
    # drop prefill tile 5: it inherits tile 4 with the step on c1
    jp = np.where(s["phase"] == 0, np.minimum((s["n_bt"].astype(np.int64) - 1) // 128, 16), -1)
    jp = np.where((s["phase"] == 0) & (s["n_bt"] > 2000), 16, jp)
    keep = jp != 5
    f2 = orc.fit_profile(*(s[k][keep] for k in ("phase", "level", "n_bt", "n_req", "n_kv", "lat_ms")), p.k, p.n_tiles,
                         p.tile_w, 1.5, Tp=p.n_ptiles, cutoff=p.prefill_cutoff)
    c5 = slice(5 * p.k, 6 * p.k)
    c4 = slice(4 * p.k, 5 * p.k)
    assert (f2["cell_status"][c5] == 1).all()
    assert np.array_equal(f2["a1"][c5], f2["a1"][c4])
    assert np.array_equal(f2["c1"][c5], f2["c1"][c4] + 1.5)


def test_pin22_single_tile_unchanged(orc):
    """T_p = 1 is the paper's single linear TTFT model: fitting with Tp = 1 equals the
    untiled fit on the same samples."""
    p = synth.make_profile("L8")
    s = profile_samples(p, 30, 8, seed=3)
    args = (s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], p.k, p.n_tiles, p.tile_w, 0.0)
    a, b = orc.fit_profile(*args), orc.fit_profile(*args, Tp=1, cutoff=123)
    for k in ("a1", "c1", "a2", "b2", "c2", "mae", "cell_status"):
        assert np.array_equal(a[k], b[k])
