"""Randomised GPU parity: many small scenarios with random layouts, ladders, SLOs, profiles,
variants and trace shapes (ties, bursts, long outputs, tiny KV capacities) in one launch,
every record byte-compared with the oracle. Complements the targeted cases of
test_gpu_parity.py / test_gpu_energy.py / test_gpu_window.py / test_gpu_noise.py."""
import numpy as np
import pytest

import synth
from synth.traces import concat_traces
from synth.workload import INF_DELTA, Layout, Slo, Workload

from test_gpu_parity import compare_records, gpu_records

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_04827_b200 as vt
    vt.lib()
    return vt


def _trace(rng, kind):
    n = int(rng.integers(0, 1500))
    if kind == 0:      # Poisson
        arr = np.cumsum(rng.exponential(1000.0 / rng.uniform(2, 60), n))
    elif kind == 1:    # integer-ms arrivals: many exact ties with event times
        arr = np.sort(rng.integers(0, 20000, n)).astype(np.float64)
    elif kind == 2:    # bursts of simultaneous arrivals
        arr = np.repeat(np.sort(rng.uniform(0, 20000, max(1, n // 20))), 20)[:n]
    else:              # dyadic times (exact sums)
        arr = np.sort(rng.integers(0, 40000, n)).astype(np.float64) / 2.0
    arr = np.sort(arr)
    inl = rng.integers(1, rng.choice([64, 2000, 9000]), n)
    outl = np.where(rng.random(n) < 0.05, 1, rng.integers(1, rng.choice([16, 300, 2500]), n))
    dur = float(arr[-1] if n else 1000.0) * rng.uniform(1.0, 1.3)
    return arr, inl.astype(np.uint32), outl.astype(np.uint32), dur


@pytest.mark.parametrize("seed", list(range(1, 11)))
def test_random_scenarios(vt, orc, seed):
    rng = np.random.default_rng(1000 + seed)
    # even seeds: untiled profiles and K <= 8 (the fast-table kernel); odd seeds: a tiled
    # profile, and every third seed ladders up to 28 levels (binary search on monotone tables)
    profiles = [synth.make_profile("L8"), synth.make_profile("B200"), synth.make_profile("Q32", n_tiles=4)]
    if seed % 2:
        profiles.append(synth.make_profile("L8", prefill_tiles=True))
    kmax = 28 if seed % 3 == 0 else 8
    grids = []
    for _ in range(8):
        k = int(rng.integers(1, kmax + 1))
        grids.append(np.sort(rng.choice(28, k, replace=False)).astype(np.uint16))
    slos = [Slo(float(rng.uniform(50, 2000)), float(rng.uniform(5, 120)), float(rng.choice([1.0, 0.9, 0.75])))
            for _ in range(16)]
    layouts = []
    for i in range(16):
        kw = dict(policy=int(rng.choice([0, 0, 1, 2])), delta_mhz=int(rng.choice([0, 150, 300, INF_DELTA])),
                  max_batch_tokens=int(rng.choice([512, 8192, 30000])),
                  kv_capacity=int(rng.choice([40000, 400000, 4000000])),
                  kv_transfer_ms=float(rng.choice([0.0, 0.0, 7.5])))
        if i >= 8:   # variants on half of the layouts
            kw.update(ctrl_mode=int(rng.integers(0, 2)), ctrl_interval_ms=float(rng.choice([0.0, 150.0, 2000.0])),
                      freq_overhead_ms=float(rng.choice([0.0, 3.0, 50.0])), itl_mode=int(rng.integers(0, 3)),
                      exec_noise=synth.exec_noise_table(float(rng.choice([0.0, 0.05, 0.2])), 256, seed=i)
                      if rng.random() < 0.5 else None)
        layouts.append(Layout(int(rng.integers(1, 9)), int(rng.integers(1, 9)), **kw))
    n_tr = 24
    traces = concat_traces([_trace(rng, t % 4) for t in range(n_tr)])
    n = 160
    scen = dict(trace_id=rng.integers(0, n_tr, n).astype(np.uint32), slo_id=rng.integers(0, 16, n).astype(np.uint32),
                layout_id=rng.integers(0, 16, n).astype(np.uint32), grid_id=rng.integers(0, 8, n).astype(np.uint32),
                profile_id=np.zeros(n, np.uint32), hash_seed=rng.integers(0, 2**63, n).astype(np.uint64))
    # profile consistent with the grid's level range (L8-grid ladders index < 28 on every profile)
    scen["profile_id"] = rng.integers(0, len(profiles), n).astype(np.uint32)
    w = Workload(f"fuzz{seed}", traces, profiles, slos, layouts, grids, scen)
    g = gpu_records(vt, w)
    o = orc.simulate_workload(w)
    compare_records(g, o)
    assert (o["status"] == 0).sum() > n // 3          # most scenarios run to completion
