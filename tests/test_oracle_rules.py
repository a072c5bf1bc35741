"""Pins of three simulator rules inside oracle_simulate that the single-decision pins (PIN-4,
PIN-5) do not reach (no GPU):

- PIN-24 backlog -> maximum frequency, as the simulator applies it at every prefill and decode
  START ("if a backlog exists, it directly selects the maximum frequency"; for decode
  S:448 "admission queue backlog (KV full) -> ... selects max frequency"). Reading A5.
- PIN-25 decode KV accounting ("each decode instance's sum of resident KV = sum over
  running requests of (input_len + 1 + tokens generated so far)") and FCFS head-of-line
  admission at iteration boundaries (readings A19, A20).
- PIN-26 the KV-transfer delay tau ("kv_transfer_ms: admission delay", "charged
  kv_transfer_ms but does not extend TTFT"): single-request closed form and FIFO order.

Nothing here re-runs the oracle's own code path to compare it with itself: the expected
batch, queue, running set, KV and level of every logged iteration are rebuilt in Python from
the trace (arrivals, lengths), the per-request times the oracle logs (first token, admission,
completion) and the rules as the paper / SPEC state them. tools/mutate_oracle.py checks that
the mutations named in VERDICT r01 (backlog forced to 0, KV release off by one, delay 2 tau)
each fail at least one of these tests.
"""

import numpy as np
import pytest

import synth
from synth.profiles import custom_profile
from synth.workload import Layout, Slo


def _lowest_ttft(p, lad, nbt, budget):
    """the lowest ladder level whose predicted TTFT (eq:pred-ttft) meets the budget;
    none -> the top (A2)."""
    for k, lv in enumerate(lad):
        if p.a1[lv] * float(nbt) + p.c1[lv] <= budget:
            return k
    return len(lad) - 1


def _lowest_itl(p, lad, n, kv, target):
    """P:380, P:387 with eq:pred-itl on the batch-size tile of N_req (A21)."""
    j = min(p.n_tiles - 1, (n - 1) // p.tile_w)
    for k, lv in enumerate(lad):
        i = j * p.k + lv
        if (p.a2[i] * float(n) + p.b2[i] * float(kv)) + p.c2[i] <= target:
            return k
    return len(lad) - 1


def _run(orc, arr, inl, outl, D, prof, slo, lay, lad, cap=200000):
    d = {}
    r = orc.simulate(np.asarray(arr, float), np.asarray(inl), np.asarray(outl), float(D), slo, lay, lad, prof,
                     7, diag=d, iter_cap=cap)
    assert r["status"] == 0
    assert len(d["iter_inst"]) < cap
    return r, d


def _heavy_trace(seed, n, rate_per_ms, in_hi, out_hi):
    rng = np.random.default_rng(seed)
    arr = np.cumsum(rng.exponential(1.0 / rate_per_ms, n))
    inl = rng.integers(1, in_hi, n)
    outl = rng.integers(1, out_hi, n)
    return arr, inl, outl


# ------------------------------------------------------------------ PIN-24 backlog (prefill)

@pytest.mark.parametrize("n_p,budget", [(1, 2000), (2, 1500), (3, 8192)])
def test_pin24_prefill_backlog_rebuilt_from_arrivals(orc, n_p, budget):
    """Every prefill START: the batch is the FCFS prefix of the instance's arrived, unbatched
    requests with sum(in) <= B (at least one, A6); backlog = an arrived request is left over
    (A5); the level is the top one iff backlog, else the lowest feasible for the waiting-time
    budget. The huge TTFT SLO makes every non-backlogged batch run at level
    0, so a dropped backlog rule changes levels, not only a flag."""
    p = synth.make_profile("L8")
    lad = [0, 6, 13, 20, 27]
    arr, inl, outl = _heavy_trace(10 + n_p, 900, 0.02 * n_p, 1200, 4)
    slo = Slo(1e7, 1e7)
    lay = Layout(n_p, 1, max_batch_tokens=budget)
    r, d = _run(orc, arr, inl, outl, arr[-1] + 1.0, p, slo, lay, lad)
    K = len(lad)
    head = list(range(n_p))                  # next unbatched request id of each instance (RR, A7)
    n_back = n_top = 0
    for e in range(len(d["iter_inst"])):
        q = int(d["iter_inst"][e])
        if q >= n_p:
            continue
        t = d["iter_start"][e]
        ids = list(range(head[q], len(arr), n_p))
        arrived = [i for i in ids if arr[i] <= t]
        assert arrived and arrived[0] == head[q]
        batch, tok = [], 0
        for i in arrived:
            if batch and tok + int(inl[i]) > budget:
                break
            batch.append(i)
            tok += int(inl[i])
        backlog = len(arrived) > len(batch)
        assert int(d["iter_load"][e]) == tok
        assert bool(d["iter_flags"][e] & 4) == backlog, (e, t)
        if backlog:
            assert int(d["iter_level"][e]) == K - 1
        else:
            bud = max(0.0, slo.ttft - (t - arr[batch[0]]))
            assert int(d["iter_level"][e]) == _lowest_ttft(p, lad, tok, bud) == 0
        # the batch's first tokens all come at the end of this iteration
        assert (d["req_tfirst"][batch] == t + d["iter_dur"][e]).all()
        n_back += backlog
        n_top += int(d["iter_level"][e]) == K - 1
        head[q] = batch[-1] + n_p
    assert all(h >= len(arr) for h in head)
    assert n_back >= 20 and n_top == n_back                 # the trace exercises the rule


# ------------------------------------------------------------------ PIN-24/25 decode

def _decode_replay(orc, p, lad, arr, inl, outl, lay, slo):
    """Rebuild every decode START from the request log and check the oracle's iteration log
    against it. Returns (#backlogged STARTs, #STARTs)."""
    r, d = _run(orc, arr, inl, outl, arr[-1] + 1.0, p, slo, lay, lad)
    n_p, K, C = lay.n_p, len(lad), lay.kv_capacity
    inl = np.asarray(inl, np.int64)
    outl = np.asarray(outl, np.int64)
    dec = d["req_decode"]
    tq, ta, td = d["req_tqueue"], d["req_tadmit"], d["req_tdone"]
    routed = outl > 1
    assert np.isnan(tq[~routed]).all() and not np.isnan(tq[routed]).any()
    assert not np.isnan(ta[routed]).any()
    # queue order: the time a request joins its instance's admission queue, then routing order
    # (FCFS across one prefill instance's batch; by prefill instance at equal times, A18)
    nb = nst = 0
    for dd in range(lay.n_d):
        mine = np.nonzero(routed & (dec == dd))[0]
        its = np.nonzero(d["iter_inst"] == n_p + dd)[0]
        starts = d["iter_start"][its]
        ends = starts + d["iter_dur"][its]
        assert (np.diff(starts) > 0).all() and (starts[1:] >= ends[:-1]).all()   # one iteration at a time
        order = sorted(mine, key=lambda i: (tq[i], (i % n_p), i))
        admitted = set()
        for e, t, t_end in zip(its, starts, ends):
            running = [i for i in mine if ta[i] < t and td[i] > t]
            # tokens generated so far = this instance's iterations started in [t_admit, t)
            gen = {i: int(((starts >= ta[i]) & (starts < t)).sum()) for i in running}
            kv = sum(int(inl[i]) + 1 + gen[i] for i in running)
            waiting = [i for i in order if tq[i] <= t and i not in admitted]
            adm = []
            for i in waiting:                                               # FCFS head of line (A20)
                if kv + int(inl[i]) + 1 > C:
                    break
                adm.append(i)
                kv += int(inl[i]) + 1
            assert sorted(adm) == sorted(i for i in mine if ta[i] == t), (dd, t)
            admitted.update(adm)
            n_req = len(running) + len(adm)
            assert int(d["iter_load"][e]) == n_req
            assert int(d["iter_kv"][e]) == kv, (dd, t, int(d["iter_kv"][e]), kv)
            # C bounds the KV only at admission (A20: "admits queued requests whose KV
            # fits"); running requests then grow by one token per iteration, so S:414's
            # "resident KV <= capacity" is not an invariant of this reading (DESIGN A20 note)
            if adm:
                assert kv <= C
            backlog = len(waiting) > len(adm)                                # A5
            assert bool(d["iter_flags"][e] & 4) == backlog
            want = K - 1 if backlog else _lowest_itl(p, lad, n_req, kv, slo.itl)
            assert int(d["iter_level"][e]) == want
            nb += backlog
            nst += 1
        # completion: the (out-1)-th iteration from admission ends at t_done (one token each)
        for i in mine:
            k = np.nonzero(starts >= ta[i])[0]
            assert len(k) >= outl[i] - 1
            assert td[i] == ends[k[outl[i] - 2]]
    return nb, nst


@pytest.mark.parametrize("n_p,n_d,cap", [(1, 1, 6000), (2, 2, 4000), (1, 3, 5000)])
def test_pin24_25_decode_backlog_and_kv_identity(orc, n_p, n_d, cap):
    """Decode STARTs on a KV-starved layout: admission is the FCFS head-of-line prefix that
    fits C; the logged N_kv equals sum over running requests of (in + 1 + generated) rebuilt
    from admission times and iteration starts; backlog = queue non-empty after
    admission, and then the level is the top one; otherwise the lowest feasible ITL
    level (level 0 under the huge ITL SLO)."""
    p = synth.make_profile("L8")
    lad = [0, 6, 13, 20, 27]
    arr, inl, outl = _heavy_trace(100 + cap, 500, 0.01, 1500, 60)
    nb, nst = _decode_replay(orc, p, lad, arr, inl, outl, Layout(n_p, n_d, kv_capacity=cap), Slo(1e7, 1e7))
    assert nb >= 20 and nst - nb >= 20


def test_pin25_kv_identity_tight_slo(orc):
    """Same replay with a realistic SLO (levels spread over the ladder) and ample KV."""
    p = synth.make_profile("L8")
    lad = [0, 6, 13, 20, 27]
    arr, inl, outl = _heavy_trace(5, 400, 0.02, 3000, 300)
    nb, nst = _decode_replay(orc, p, lad, arr, inl, outl, Layout(2, 2), Slo(600, 45))
    assert nst > 100


# ------------------------------------------------------------------ PIN-26 KV-transfer delay

def _lin(K=1, a1=0.25, c1=10.0, a2=0.5, b2=0.001, c2=20.0):
    z = np.ones(K)
    return custom_profile([1005 + 15 * i for i in range(K)], a1 * z, c1 * z, a2 * z, b2 * z, c2 * z,
                          np.full(2 * K, 100.0))


@pytest.mark.parametrize("tau", [0.0, 12.5, 1000.0])
def test_pin26_single_request_transfer_delay(orc, tau):
    """1P1D, one request at t = 0 on a one-level, one-tile profile:
    t_first = TT = a1*in + c1 (independent of tau), the request joins the admission
    queue at t_first + tau, is admitted there (decode idle), and iteration j = 0..out-2
    runs at (N_req = 1, N_kv = in + 1 + j): t_done = t_first + tau + sum_j (a2 + b2 (in+1+j) + c2)."""
    p = _lin()
    inl, outl = 300, 41
    r, d = _run(orc, [0.0], [inl], [outl], 0.0, p, Slo(1e6, 1e6), Layout(1, 1, kv_transfer_ms=tau), [0])
    tt = 0.25 * inl + 10.0
    assert d["req_tfirst"][0] == tt and r["sum_ttft_ms"] == tt
    assert d["req_tqueue"][0] == tt + tau and d["req_tadmit"][0] == tt + tau
    itl_sum = sum(0.5 + 0.001 * (inl + 1 + j) + 20.0 for j in range(outl - 1))
    assert abs(d["req_tdone"][0] - (tt + tau + itl_sum)) <= 1e-12 * (tt + tau + itl_sum)
    mean = (tau + itl_sum) / (outl - 1)
    assert abs(r["sum_itl_mean_ms"] - mean) <= 1e-12 * mean
    # the decode instance is idle during the transfer: busy decode time = sum of ITLs only
    assert abs(r["busy_ms_decode"] - itl_sum) <= 1e-12 * itl_sum
    assert r["horizon_ms"] == d["req_tdone"][0]


def test_pin26_transfer_fifo_and_capacity(orc):
    """Two requests batched together (same t_first) reach the admission queue together at
    t_first + tau in FCFS order; with room for only one, the first is admitted at once and the
    second at the START that follows the first one's completion. With 2 prefill instances the
    request whose prefill ends first reaches decode first, whatever its id."""
    tau = 7.5
    p = _lin()
    inl = [100, 100]
    r, d = _run(orc, [0.0, 0.0], inl, [5, 3], 0.0, p, Slo(1e6, 1e6),
                Layout(1, 1, kv_transfer_ms=tau, kv_capacity=150), [0])
    tt = 0.25 * 200 + 10.0
    assert (d["req_tfirst"] == tt).all() and (d["req_tqueue"] == tt + tau).all()
    assert d["req_tadmit"][0] == tt + tau
    assert d["req_tadmit"][1] == d["req_tdone"][0] > tt + tau
    its = lambda kv0, n: sum(0.5 + 0.001 * (kv0 + j) + 20.0 for j in range(n))
    assert abs(d["req_tdone"][0] - (tt + tau + its(101, 4))) <= 1e-12 * d["req_tdone"][0]
    assert abs(d["req_tdone"][1] - (d["req_tadmit"][1] + its(101, 2))) <= 1e-12 * d["req_tdone"][1]
    # 2P1D: request 0 (long prompt, prefill 0) finishes after request 1 (short, prefill 1)
    r, d = _run(orc, [0.0, 0.0], [2000, 40], [5, 200], 0.0, p, Slo(1e6, 1e6),
                Layout(2, 1, kv_transfer_ms=tau, kv_capacity=2001 + 1), [0])
    t0, t1 = 0.25 * 2000 + 10.0, 0.25 * 40 + 10.0
    assert d["req_tfirst"][0] == t0 and d["req_tfirst"][1] == t1
    assert d["req_tqueue"][1] == t1 + tau and d["req_tadmit"][1] == t1 + tau
    assert d["req_tqueue"][0] == t0 + tau and d["req_tadmit"][0] > t0 + tau     # waits: KV held by 1
    assert d["req_tadmit"][0] == d["req_tdone"][1]
