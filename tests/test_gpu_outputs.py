"""GPU parity of voltana_simulate_ex's optional outputs (DESIGN.md
E1-E3): per-request records and per-instance iteration time series, element by element
against the oracle's diagnostics (the oracle's global iteration log regrouped per instance)."""
import dataclasses

import numpy as np
import pytest

import synth
from synth.workload import Layout, Slo, POLICY_ENERGY

from test_gpu_parity import compare_records

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_04827_b200 as vt
    vt.lib()
    return vt


def _oracle_scenario(orc, w, c, iter_cap):
    s = w.scen
    a, ii, o, D = w.traces.trace(int(s["trace_id"][c]))
    lay = w.layouts[s["layout_id"][c]]
    d = {}
    r = orc.simulate(a, ii, o, D, w.slos[s["slo_id"][c]], lay, w.grids[s["grid_id"][c]],
                     w.profiles[s["profile_id"][c]], int(s["hash_seed"][c]), diag=d, iter_cap=iter_cap)
    return r, d, lay, o


def _check(vt, orc, w, requests=True, cap=1 << 20):
    dw = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
    outs = dw.outputs(requests=requests, iter_cap=cap)
    dw.launch(outputs=outs)
    g = dw.records()
    mask = np.ones(w.n, bool) if requests is True else np.asarray(requests, bool)
    n_req = n_it = 0
    for c in range(w.n):
        r, d, lay, outl = _oracle_scenario(orc, w, c, 1 << 22)
        compare_records(g[c:c + 1], np.array([r]))
        if mask[c]:
            q = outs.requests(c)
            dec = np.where(d["req_decode"] < 0, 0xFF, d["req_decode"]).astype(np.uint8)
            cse = np.where(d["req_decode"] < 0, 0xFF, d["req_case"]).astype(np.uint8)
            assert np.array_equal(q["tfirst"], d["req_tfirst"])
            assert np.array_equal(q["tdone"], d["req_tdone"])
            assert np.array_equal(q["itl"], d["req_itl"])
            assert np.array_equal(q["decode"], dec)
            assert np.array_equal(q["case"], cse)
            n_req += len(q["tfirst"])
        else:
            with pytest.raises(KeyError):
                outs.requests(c)
        per, cnt = outs.iterations(c)
        assert np.array_equal(cnt, d["iters"].astype(np.int64))
        for u, arr in enumerate(per):
            m = d["iter_inst"] == u
            k = min(int(m.sum()), cap)
            assert len(arr) == k
            assert np.array_equal(arr["t_start"], d["iter_start"][m][:k])
            assert np.array_equal(arr["dur_ms"], d["iter_dur"][m][:k])
            assert np.array_equal(arr["level"], d["iter_level"][m][:k])
            assert np.array_equal(arr["load"], d["iter_load"][m][:k])
            assert np.array_equal(arr["n_kv"], d["iter_kv"][m][:k])
            assert np.array_equal(arr["flags"], d["iter_flags"][m][:k])
            n_it += k
    return n_req, n_it


def test_outputs_c1_full(vt, orc):
    n_req, n_it = _check(vt, orc, synth.build_config("C1"))
    assert n_req == 200 and n_it > 1000


@pytest.mark.parametrize("kw", [dict(), dict(ctrl_interval_ms=400.0, freq_overhead_ms=50.0),
                                dict(policy=POLICY_ENERGY, exec_noise=synth.exec_noise_table(0.1, 512))])
def test_outputs_c3_variants(vt, orc, kw):
    w = synth.build_config("C3", scenarios=list(range(0, 256, 29)), duration_scale=0.1)
    w = dataclasses.replace(w, layouts=[dataclasses.replace(x, **kw) for x in w.layouts])
    mask = np.arange(w.n) % 2 == 0
    n_req, n_it = _check(vt, orc, w, requests=mask)
    assert n_req > 0 and n_it > 0


def test_outputs_truncated_series(vt, orc):
    w = synth.build_config("C4", scenarios=[3, 700, 4000], duration_scale=0.05)
    _check(vt, orc, w, requests=True, cap=16)


def test_outputs_do_not_change_records(vt, orc):
    w = synth.build_config("C4", scenarios=list(range(0, 4096, 409)), duration_scale=0.1)
    base = vt.simulate(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
    dw = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
    dw.launch(outputs=dw.outputs(requests=True, iter_cap=64))
    assert dw.records().tobytes() == base.tobytes()


@pytest.mark.parametrize("sigma", [0.0, 0.05])
def test_fit_simulate_loop(vt, orc, sigma):
    """K4 series -> K5 samples -> K1 fit equals the oracle fit of the oracle's iteration log
    (same samples in another order: within 1e-12), and the loop's profile drives K4 again."""
    from test_oracle_loop import log_samples
    w = synth.build_config("C4", scenarios=list(range(3584, 4096, 64)), duration_scale=0.3)
    if sigma > 0:
        w = dataclasses.replace(w, layouts=[dataclasses.replace(x, exec_noise=synth.exec_noise_table(sigma, 4096))
                                            for x in w.layouts])
    p = w.profiles[0]
    dw = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
    outs = dw.outputs(iter_cap=1 << 14)
    dw.launch(outputs=outs)
    smp = outs.samples(profile_id=0)
    fit = vt.fit_profile(smp["phase"], smp["level"], smp["n_bt"], smp["n_req"], smp["n_kv"], smp["lat_ms"],
                         p.k, p.n_tiles, p.tile_w, 0.0)
    torch.cuda.synchronize()
    cols = []
    for c in range(w.n):
        r, d, lay, _ = _oracle_scenario(orc, w, c, 1 << 22)
        cols.append(log_samples(d, w.grids[w.scen["grid_id"][c]], lay.n_p))
    osmp = [np.concatenate([x[i] for x in cols]) for i in range(6)]
    ref = orc.fit_profile(*osmp, p.k, p.n_tiles, p.tile_w, 0.0)
    st = fit["cell_status"].cpu().numpy()
    assert (st == ref["cell_status"]).all()
    n_valid = int((smp["phase"] <= 1).sum().item())
    assert n_valid == len(osmp[0])
    assert int(fit["invalid"].cpu().numpy().view(np.uint64)[0]) == smp["phase"].numel() - n_valid
    ok = st == 0
    K = p.k
    for name, sl in (("a1", slice(0, K)), ("c1", slice(0, K)), ("a2", slice(K, None)), ("b2", slice(K, None)),
                     ("c2", slice(K, None))):
        g = fit[name].cpu().numpy()
        o = ref[name]
        m = ok[sl]
        err = np.abs(g[m] - o[m]) / np.maximum(np.abs(o[m]), 1e-9)
        assert err.max() <= 1e-12 or np.abs(g[m] - o[m]).max() < 1e-12, (name, err.max())
    # close the loop: the fitted profile drives the simulator again (ladder [0]: the level whose
    # ITL cells the log covered), GPU and oracle on the same fitted tables
    dp2 = vt.DeviceProfile.from_fit(fit, p.mhz, p.dyn, p.p_idle, p.tdp, p.u_half_prefill, p.u_half_decode,
                                    p.n_tiles, p.tile_w)
    host = {k: fit[k].cpu().numpy() for k in ("a1", "c1", "a2", "b2", "c2")}
    p2 = dataclasses.replace(p, **host)
    w2 = dataclasses.replace(w, grids=[np.array([0], np.uint16)], profiles=[p2],
                             scen=dict(w.scen, grid_id=np.zeros(w.n, np.uint32)))
    g2 = vt.simulate(w2.traces, w2.slos, w2.layouts, w2.grids, [dp2], w2.scen)
    compare_records(g2, orc.simulate_workload(w2))
    assert (g2["status"] == 0).all()
