"""PIN-15: the seeded input generators (not the method)."""

import numpy as np

import synth
from synth.traces import DATASETS, TraceSpec, gen_trace, lognormal_params


def test_lognormal_moments_appendix_a():
    """Moment matching to tab:length_statistics:
    10^6 draws recover mean/std within 2% (pre-truncation targets)."""
    rng = np.random.default_rng(0)
    for ds in ("SG", "LM"):
        for which in ("in", "out"):
            mean, std = DATASETS[ds][which]
            mu, sig = lognormal_params(mean, std)
            x = rng.lognormal(mu, sig, 10**6)
            assert abs(x.mean() / mean - 1) < 0.02 and abs(x.std() / std - 1) < 0.02, (ds, which)


def test_poisson_count_and_lengths():
    a, i, o, D = gen_trace(TraceSpec("SG", "poisson", 100.0, lam=10.0, key=(0, 0, 1)))
    assert abs(len(a) - 1000) < 3 * np.sqrt(1000)
    assert D == 100000.0 and (np.diff(a) >= 0).all() and a[-1] < D
    assert i.min() >= 1 and o.min() >= 1 and i.max() <= 32768 and o.max() <= 32768
    a2, i2, o2, _ = gen_trace(TraceSpec("SG", "poisson", 100.0, lam=10.0, key=(0, 0, 1)))
    assert (a == a2).all() and (i == i2).all() and (o == o2).all()  # seeded determinism


def test_sharegpt_like_trace_means():
    a, i, o, _ = gen_trace(TraceSpec("SG", "poisson", 600.0, lam=40.0, key=(0, 0, 2)))
    assert abs(i.mean() / 280.27 - 1) < 0.06 and abs(o.mean() / 190.90 - 1) < 0.06


def test_mmpp_time_average_rate():
    a, *_ = gen_trace(TraceSpec("LM", "mmpp", 3000.0, lam=20.0, key=(0, 0, 3)))
    assert abs(len(a) / 3000.0 / 20.0 - 1) < 0.15                   # time-average = lam-bar
    # bursty: the count over 10-s windows is over-dispersed vs Poisson (variance > mean)
    c = np.bincount((a // 10000).astype(int))
    assert c.var() > 2 * c.mean()


def test_phased_pd_mix_alternates():
    a, i, o, _ = gen_trace(TraceSpec("SG", "phased", 1200.0, lam=8.0, key=(0, 0, 4)))
    seg = (a // 300000).astype(int)
    r = [i[seg == s].mean() / o[seg == s].mean() for s in range(4)]
    assert r[0] > 2 * r[1] and r[2] > 2 * r[3]                       # P/D ratio flips


def test_piecewise_rates():
    a, *_ = gen_trace(TraceSpec("SG", "piecewise", 1200.0, rates=(2.0, 8.0), key=(0, 0, 5)))
    seg = np.bincount((a // 300000).astype(int), minlength=4)
    assert seg[1] > 2.5 * seg[0] and seg[3] > 2.5 * seg[2]


def test_profiles_anchors():
    p = synth.make_profile("L8")
    assert p.k == 28 and p.mhz[0] == 1005 and p.mhz[-1] == 1410      # A27 grid
    for f in (1005, 1095, 1200, 1305, 1410):                           # P:600, P:692 ladders on grid
        p.level_of(f)
    # coefficient-monotone (A32): non-increasing in f within every tile
    for arr in (p.a1, p.c1):
        assert (np.diff(arr) <= 0).all()
    for arr in (p.a2, p.b2, p.c2):
        assert (np.diff(arr.reshape(p.n_tiles, p.k), axis=1) <= 0).all()
    b = synth.make_profile("B200")
    assert b.k == 60 and b.mhz[-1] == 1965


def test_configs_shapes():
    for name, n in (("C1", 1), ("C2", 1024), ("C3", 256), ("C4", 4096), ("C5", 16384)):
        w = synth.build_config(name, scenarios=[0])
        assert w.n == 1
    w = synth.build_config("C1")
    assert w.n == 1 and w.traces.lengths()[0] == 200
