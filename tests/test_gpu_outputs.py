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
