"""PIN-23: per-request ITL aggregation modes for attainment (SPEC.md:565 `itl_mode` {Mean, Max,
P99}; E3). Mean is the paper-facing default (A30); Max is the largest
inter-token gap of the request; P99 is the nearest-rank 99th percentile of its out - 1 gaps.

Pins: a closed-form single-request trace whose three modes disagree in a known way, the
nearest-rank boundary at n = 100 / 101 gaps, invariants on random workloads, and a
re-derivation of every request's gaps from the iteration log compared with numpy's
inverted-CDF percentile.
"""
import numpy as np
import pytest

import synth
from synth.profiles import custom_profile
from synth.workload import Layout, Slo


def _flat(c=20.0):
    K = 2
    z = np.zeros(K)
    return custom_profile([1005, 1410], z, np.array([100.0, 60.0]), z, z, np.array([c, c / 2]),
                          np.array([100.0, 200.0, 50.0, 90.0]), p_idle=60.0, tdp=1e9)


@pytest.mark.parametrize("out", [102, 101, 51, 11, 10])
def test_pin23_single_request_modes(orc, out):
    """Gaps [ov + c, c, ..., c] (n = out - 1 of them; c = 20 ms constant ITL, ov = 50 ms blocking
    frequency set at the first decode iteration, C3), SLO 25 ms:
      mean (ov + n c) / n <= 25  iff n >= 10;
      max  = ov + c = 70 > 25    never;
      P99  = the ceil(0.99 n)-th smallest: c when ceil(0.99 n) <= n - 1, i.e. n >= 100."""
    p = _flat()
    slo = Slo(1e6, 25.0)
    n = out - 1
    expect = {0: int(n >= 10), 1: 0, 2: int(n >= 100)}
    for mode in (0, 1, 2):
        r = orc.simulate(np.array([0.0]), [100], [out], 0.0, slo, Layout(1, 1, freq_overhead_ms=50.0, itl_mode=mode),
                         np.array([0, 1], np.uint16), p)
        assert int(r["n_itl_ok"]) == expect[mode], (out, mode)
        assert r["sum_itl_mean_ms"] == (50.0 + n * 20.0) / n     # the report sum stays the mean (E3)


def test_pin23_modes_agree_without_overhead(orc):
    """Constant gaps (no overhead, constant ITL): mean = max = P99 for every request."""
    p = _flat()
    rng = np.random.default_rng(23)
    arr = np.sort(rng.uniform(0, 1000, 30))
    outl = rng.integers(2, 300, 30)
    res = [orc.simulate(arr, np.full(30, 50), outl, 0.0, Slo(1e6, 20.0), Layout(1, 1, itl_mode=m),
                        np.array([0], np.uint16), p) for m in (0, 1, 2)]
    assert res[0]["n_itl_ok"] == res[1]["n_itl_ok"] == res[2]["n_itl_ok"]


def _gaps_from_log(d, n_p, tfirst, tdone, dec, outl, ov):
    """Re-derive each request's token gaps from the iteration log: the tokens of a request on
    decode instance u are the END times of u's consecutive iterations ending at t_done."""
    ends = {}
    for inst, t0, dur, fl in zip(d["iter_inst"], d["iter_start"], d["iter_dur"], d["iter_flags"]):
        if inst >= n_p:
            ends.setdefault(int(inst) - n_p, []).append((t0 + ov if fl & 2 else t0) + dur)
    out = {}
    for i in range(len(outl)):
        if outl[i] < 2:
            continue
        e = ends[int(dec[i])]
        f = e.index(tdone[i])
        a = f - (int(outl[i]) - 2)
        g = [e[a] - tfirst[i]] + [e[j] - e[j - 1] for j in range(a + 1, f + 1)]
        assert len(g) == outl[i] - 1
        out[i] = np.array(g)
    return out


@pytest.mark.parametrize("ov,interval", [(0.0, 0.0), (50.0, 0.0), (3.0, 300.0)])
def test_pin23_rederived_from_the_iteration_log(orc, ov, interval):
    p = synth.make_profile("L8")
    rng = np.random.default_rng(230)
    m = 150
    arr = np.sort(rng.uniform(0, 8000, m))
    inl = rng.integers(20, 2500, m)
    outl = rng.integers(1, 400, m)
    lad = np.array([0, 6, 13, 20, 27], np.uint16)
    slo = Slo(600.0, 30.0)
    counts = {}
    for mode in (0, 1, 2):
        d = {}
        lay = Layout(2, 2, freq_overhead_ms=ov, ctrl_interval_ms=interval, itl_mode=mode)
        r = orc.simulate(arr, inl, outl, 8000.0, slo, lay, lad, p, diag=d, iter_cap=400000)
        assert r["status"] == 0
        counts[mode] = int(r["n_itl_ok"])
    gaps = _gaps_from_log(d, 2, d["req_tfirst"], d["req_tdone"], d["req_decode"], outl, ov)
    n1 = int((outl == 1).sum())
    mean_ok = sum(1 for i, g in gaps.items() if (d["req_tdone"][i] - d["req_tfirst"][i]) / (outl[i] - 1) <= 30.0)
    max_ok = sum(1 for g in gaps.values() if g.max() <= 30.0)
    p99_ok = sum(1 for g in gaps.values() if np.percentile(g, 99, method="inverted_cdf") <= 30.0)
    assert counts[0] == n1 + mean_ok
    assert counts[1] == n1 + max_ok
    assert counts[2] == n1 + p99_ok
    assert counts[1] <= counts[2] and counts[1] <= counts[0]
    if ov > 0:
        assert counts[1] < counts[0]                    # the overhead gaps are visible to Max only
