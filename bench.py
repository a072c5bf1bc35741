#!/usr/bin/env python
"""Benchmark: scenario-steps/sec (EcoFreq controller + EcoRoute router decisions) of the
batched VoltanaLLM policy evaluation on B200 (BASELINE.json metric).

Default workload (BASELINE configs[3], "SLO x arrival-rate x seed sweep, 4096 scenarios"): C4 —
4096 scenarios = 4 SLO x 8 Poisson rates x 128 seeds, 2P2D, 5-level ladder, Delta = 150,
LLaMA-3.1-8B-shaped profile, ShareGPT-like synthetic traces of 600 s. `--config C2|C3|C5`
selects the other BASELINE sweeps (C1 is the oracle-sized single scenario).

One step = one pass of the whole hot path: K1 fits the EcoPred profile from 2M synthetic
profiling samples, then K4 simulates every scenario with the fitted tables (every controller
and router decision, energy integration, per-scenario records); for N > 1 the records are
all-gathered over NCCL inside the step.

Multi-GPU (one process per GPU): `--gpus N` without a torchrun environment re-launches itself
under torch.distributed.run. `--scaling weak` (default): rank r sweeps its own seed block of the
config. `--scaling strong`: the one fixed sweep is split by the deterministic LPT partition
(shard.lpt_partition) and the gathered records are placed back in global scenario order.

Same-run correctness gate: after the warm-up, the CPU oracle (test infrastructure) runs on the
same fitted tables and the same scenarios (all of them when that is <= ~30 core-seconds, else a
stratified sample plus the 8 heaviest); decision counters and hashes must be identical and fp64
totals within 1e-9 relative, else the line reports `parity.ok = false` and the exit status is 1.
That oracle run, timed on the host cores, is the `cpu_baseline` (N = 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]
                    [--scaling weak|strong]
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scenario-steps/sec (ctrl+router decisions) at 1/2/4/8 B200; % of HBM roofline"  # BASELINE.json
UNIT = "steps/s"
N_SAMPLES = 2_000_000
NODE_BYTES = 16            # K4b's per-request input (one node: t_first, in, out, next) = trace bytes
RECORD_BYTES = 128
ORACLE_BUDGET = 4.0e8      # decisions the parity oracle may simulate (~30 core-seconds)
INT_FIELDS = ("status", "n_requests", "n_ttft_ok", "n_itl_ok", "n_both_ok", "prefill_iters", "steps_ctrl",
              "steps_route", "decision_hash")
FP_FIELDS = ("sum_ttft_ms", "sum_itl_mean_ms", "e_prefill_busy_j", "e_prefill_idle_j", "e_decode_busy_j",
             "e_decode_idle_j", "busy_ms_prefill", "busy_ms_decode", "top_level_ms", "horizon_ms")

WORKLOADS = {
    "C1": "C1: 1 trace, 1P1D, 3 levels [1005,1200,1410] MHz, linear latency model (T=1), 200 ShareGPT-like requests",
    "C2": "C2: 1024 scenarios = 8 Poisson rates x 128 seeds, 1P1D, 28-level A100 grid 1005..1410 MHz, "
          "LLaMA-3.1-8B-shaped profile, ShareGPT-like traces of 600 s",
    "C3": "C3: 256 scenarios = 2 ladders x 4 time-varying patterns x 32 seeds, 2P2D EcoRoute, Qwen-32B-shaped "
          "profile, SLO 1200/120, ShareGPT-like traces of 1200 s",
    "C4": "C4: 4096 scenarios = 4 SLO x 8 Poisson rates x 128 seeds, 2P2D, 5-level ladder [1005..1410] MHz, "
          "Delta=150, LLaMA-3.1-8B-shaped profile, ShareGPT-like traces of 600 s",
    "C5": "C5: 16384 scenarios = 4 SLO x 16 rates x 256 seeds, 4P4D, 60-level B200 grid 1080..1965 MHz, "
          "Delta=150, B200-style profile, bursty LMSYS-like MMPP-2 traces of 300 s",
}
REF_PER_STEP = {"C1": 1, "C2": 1024, "C3": 256, "C4": 1024, "C5": 128}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the oracle timing (parity still runs)")
    ap.add_argument("--no-parity", action="store_true", help="skip the same-run oracle check (profiling runs only)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-streaming", action="store_true", help="skip the K1/K2/K3 streaming and variant sub-benches")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo check of the multi-rank plumbing (spawn, partition, record gather); no GPU work")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args) -> int:
    """--gpus N outside torchrun: re-run this script under torch.distributed.run, one rank per
    GPU (127.0.0.1 rendezvous). Rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def workload_config(args, world):
    par = (f"scenario-sharded x{world} (weak: one seed block per GPU)" if args.scaling == "weak"
           else f"scenario-sharded x{world} (strong: one sweep, LPT partition)")
    return {"workload": WORKLOADS[args.config], "config_id": args.config, "scaling": args.scaling,
            "l2": "flushed between timed steps (256 MiB write); inputs > L2 (C2-C5)", "parallelism": par}


def build_shard(args, rank, world):
    """The rank's scenarios: (workload, global indices of its scenarios in caller order, parts)."""
    import synth
    from paper_2509_04827_b200.shard import lpt_partition, scenario_costs, weak_parts
    if args.scaling == "weak" or world == 1:
        w = synth.build_config(args.config, seed_block=rank)
        parts = weak_parts(w.n, world)
        return w, parts
    full = synth.build_config(args.config, seed_block=0)
    parts = lpt_partition(scenario_costs(full), world)
    return full.subset(parts[rank]), parts


def fit_samples(prof):
    """2 M calibration samples in recording order (one profiling run per frequency level, P:503;
    DESIGN.md §4)."""
    from synth.samples import profile_samples
    m = max(2, N_SAMPLES // (prof.k * (1 + prof.n_tiles)))
    return profile_samples(prof, m, m, noise_sigma=0.02, seed=0, shuffle=False)


def fitted_host_profile(prof, fit):
    """The profile the GPU simulated with: the generating profile's grid and power tables with
    the K1-fitted EcoPred coefficients (copied D2H once) — the oracle's input for parity."""
    g = {k: fit[k].cpu().numpy().astype(np.float64).copy() for k in ("a1", "c1", "a2", "b2", "c2")}
    return dataclasses.replace(prof, **g)


# ---------------------------------------------------------------------------- oracle (CPU)
_ORC_W = None


def _orc_init():
    import oracle
    oracle.lib()


def _orc_run(task):
    import oracle
    idx, prof = task
    w = _ORC_W if prof is None else dataclasses.replace(_ORC_W, profiles=[prof])
    t0 = time.perf_counter()
    r = oracle.simulate_workload(w, idx)
    return r, time.perf_counter() - t0


class OraclePool:
    """The oracle on `cores` forked processes (test infrastructure: parity and the CPU baseline)."""

    def __init__(self, w, cores):
        import multiprocessing as mp
        global _ORC_W
        _ORC_W = w
        self.cores = cores
        self.pool = mp.get_context("fork").Pool(cores, initializer=_orc_init)
        self.pool.map(_orc_run, [([0], None)] * cores)            # warm the workers

    def run(self, idx, prof=None):
        """Records for scenarios idx (in that order) and the wall time."""
        idx = np.asarray(idx, np.int64)
        # interleaved chunks: the cost-ordered sample spreads evenly over the workers
        nch = max(1, min(len(idx), self.cores * 8))
        chunks = [idx[c::nch] for c in range(nch)]
        t0 = time.perf_counter()
        res = self.pool.map(_orc_run, [(c, prof) for c in chunks])
        wall = time.perf_counter() - t0
        out = np.zeros(len(idx), res[0][0].dtype)
        for c, (r, _) in enumerate(res):
            out[c::nch] = r
        return out, wall

    def close(self):
        self.pool.close()
        self.pool.join()


def parity_sample(rec, n_budget=ORACLE_BUDGET, min_sample=32, n_heavy=8):
    """All scenarios when the oracle can redo the sweep within the budget, else a stratified
    sample (every k-th) plus the n_heavy heaviest (most decisions)."""
    steps = (rec["steps_ctrl"] + rec["steps_route"]).astype(np.float64)
    n = len(steps)
    if steps.sum() <= n_budget:
        return np.arange(n), f"all {n} scenarios"
    k = max(1, int(math.ceil(steps.sum() / n_budget)))
    heavy = np.argsort(-steps, kind="stable")[:n_heavy]
    idx = np.unique(np.concatenate([np.arange(0, n, k), heavy]))
    if len(idx) < min_sample:
        idx = np.unique(np.concatenate([idx, np.linspace(0, n - 1, min_sample).astype(np.int64)]))
    return idx, f"{len(idx)} of {n} scenarios (every {k}th + the {n_heavy} heaviest)"


def compare(gpu, orc):
    ints_ok = all(bool((gpu[f] == orc[f]).all()) for f in INT_FIELDS)
    rel = 0.0
    for f in FP_FIELDS:
        g, o = gpu[f].astype(np.float64), orc[f].astype(np.float64)
        e = np.abs(g - o) / np.maximum(np.abs(o), 1e-300)
        rel = max(rel, float(e.max()) if len(e) else 0.0)
    exact = int((gpu.view(np.uint8).reshape(len(gpu), 128) == orc.view(np.uint8).reshape(len(orc), 128))
                .all(axis=1).sum()) if len(gpu) else 0
    return {"checked": int(len(gpu)), "bitexact": exact, "int_fields_equal": ints_ok, "max_rel_err_fp64": rel,
            "decisions_gpu": int((gpu["steps_ctrl"] + gpu["steps_route"]).sum()),
            "decisions_oracle": int((orc["steps_ctrl"] + orc["steps_route"]).sum()),
            "ok": bool(ints_ok and rel <= 1e-9)}


# ---------------------------------------------------------------------------- clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        """Start sampling every 100 ms and return once the first sample is written (so the timed
        region that follows is covered from its start)."""
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
            return
        t0 = time.time()
        while time.time() - t0 < 10.0 and self.p.poll() is None:
            self.f.flush()
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.05)
        self.skip = len(open(self.f.name).read().strip().splitlines())   # samples taken before the region

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        lines = open(self.f.name).read().strip().splitlines()
        lines = lines[getattr(self, "skip", 0):] or lines[-1:]       # the timed region's samples
        rows = [r.split(",") for r in lines if r.count(",") >= 8]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


# ---------------------------------------------------------------------------- sub-benches (rank 0)
def streaming_kernels(vt, torch, dev, hbm_gbs, reps=100):
    """K2 control_step, K3 route_batch and K1 fit_profile on large SoA batches (HBM-bound):
    algorithmic bytes per launch / mean CUDA-event time, against the measured copy bandwidth."""
    import synth
    from synth.samples import profile_samples
    prof = synth.make_profile("L8")
    dp = vt.DeviceProfile(prof, dev)
    lad = [0, 6, 13, 20, 27]
    g = torch.Generator(device=dev).manual_seed(0)
    n = 1 << 25
    u32 = lambda lo, hi, size: torch.randint(lo, hi, size, generator=g, device=dev, dtype=torch.int64).to(torch.int32).view(torch.uint32)
    load = u32(1, 700, (n,))
    kv = u32(700, 300000, (n,))
    q = (torch.rand(n, generator=g, device=dev) < 0.05).to(torch.int32).view(torch.uint32)
    tgt = torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 60 + 20
    out = {}

    def timed(fn):
        for _ in range(20):                     # warm-up: clocks and caches settle
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps / 1000.0

    s = timed(lambda: vt.control_step(dp, 1, lad, load, kv, q, None, tgt))
    by = n * (4 + 4 + 4 + 8 + 2 + 1)
    out["control_step"] = {"items": n, "bytes_per_item": 23, "ms": s * 1e3, "achieved_gbs": by / s / 1e9,
                           "frac": by / s / 1e9 / hbm_gbs, "decisions_per_s": n / s}
    nd, m = 2, 1 << 24
    nr = u32(0, 500, (m * nd,))
    nk = u32(500, 200000, (m * nd,))
    rin = u32(1, 4000, (m,))
    cur = torch.zeros(m, dtype=torch.int32, device=dev).view(torch.uint32)
    s = timed(lambda: vt.route_batch(dp, lad, nd, nr, nk, rin, tgt[:m], 150, 0, cur))
    by = m * (8 * nd + 4 + 8 + 4 + 4 + 2 + 1 + 1)
    out["route_batch"] = {"items": m, "bytes_per_item": 8 * nd + 24, "ms": s * 1e3, "achieved_gbs": by / s / 1e9,
                          "frac": by / s / 1e9 / hbm_gbs, "decisions_per_s": m / s}
    # samples in the order a profiling run records them (one run per frequency level,
    # iterations in time order, batch sizes drifting: cell-clustered); "_shuffled" is the
    # adversarial order (random cells in every 32-sample chunk)
    # (runs of 4201 / 32771 samples per cell: cell boundaries fall inside 128-sample chunks)
    for label, per_cell, shuffled in (("fit_profile", 4201, False), ("fit_profile_large", 32771, False),
                                      ("fit_profile_large_shuffled", 32771, True)):
        smp = profile_samples(prof, per_cell, per_cell, noise_sigma=0.02, seed=9, shuffle=shuffled)
        to = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else
                                        (a.view(np.int16) if a.dtype == np.uint16 else a)).to(dev)
        d = {k: to(v) for k, v in smp.items()}
        for k in ("n_bt", "n_req", "n_kv"):
            d[k] = d[k].view(torch.uint32)
        d["level"] = d["level"].view(torch.uint16)
        ns = int(d["lat_ms"].numel())
        fo = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, prof.n_tiles)
        s = timed(lambda: vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k,
                                         prof.n_tiles, workspace=fo["workspace"], out=fo))
        by = 3 * ns * 23
        out[label] = {"samples": ns, "bytes_per_sample": 69, "ms": s * 1e3, "achieved_gbs": by / s / 1e9,
                      "frac": by / s / 1e9 / hbm_gbs, "note": "3 streaming passes x 23 B/sample"}
        if label == "fit_profile_large":   # ~10^8 samples: the recording-order runs repeated 6 times
            d6 = {k: v.repeat(6) for k, v in d.items()}
            ns6 = int(d6["lat_ms"].numel())
            fo6 = vt.fit_profile(d6["phase"], d6["level"], d6["n_bt"], d6["n_req"], d6["n_kv"], d6["lat_ms"], prof.k,
                                 prof.n_tiles)
            s = timed(lambda: vt.fit_profile(d6["phase"], d6["level"], d6["n_bt"], d6["n_req"], d6["n_kv"],
                                             d6["lat_ms"], prof.k, prof.n_tiles, workspace=fo6["workspace"], out=fo6))
            by = 3 * ns6 * 23
            out["fit_profile_xl"] = {"samples": ns6, "bytes_per_sample": 69, "ms": s * 1e3,
                                     "achieved_gbs": by / s / 1e9, "frac": by / s / 1e9 / hbm_gbs,
                                     "note": "3 streaming passes x 23 B/sample; recording order, 6 runs per cell"}
            del d6, fo6
        del d, fo
    return out


def variant_kernels(vt, torch, w, dprof, dev, reps=3):
    """K4 on the same sweep with each §8(f) variant switched on for every scenario (the
    variant instantiation): mean CUDA-event time of one launch and decisions/s. Context for
    what the variants cost; the headline line is the paper's policies."""
    import synth
    variants = {
        "energy_router+energy_ctrl": dict(policy=2, ctrl_mode=1),
        "window_300ms+overhead_3ms": dict(ctrl_interval_ms=300.0, freq_overhead_ms=3.0),
        "exec_noise_sigma_0.05": dict(exec_noise=synth.exec_noise_table(0.05, 4096)),
        "itl_p99": dict(itl_mode=2),
    }
    out = {}
    for name, kw in variants.items():
        lays = [dataclasses.replace(x, **kw) for x in w.layouts]
        wl = vt.DeviceWorkload(w.traces, w.slos, lays, w.grids, [dprof], w.scen, device=dev)
        wl.launch()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            wl.launch()
        b.record()
        b.synchronize()
        rec = wl.records()
        steps = int((rec["steps_ctrl"] + rec["steps_route"]).sum())
        ms = a.elapsed_time(b) / reps
        out[name] = {"simulate_ms": ms, "decisions": steps, "decisions_per_s": steps / (ms / 1000.0)}
        del wl
    return out


def heavy_alone(vt, torch, w, dprof, rec, dev, counts=(1, 148), reps=3):
    """The strong-scaling bound: the heaviest scenarios of this rank simulated alone (one warp
    each on an otherwise idle GPU) — the length of the longest serial decision chain."""
    steps = (rec["steps_ctrl"] + rec["steps_route"]).astype(np.int64)
    order = np.argsort(-steps, kind="stable")
    out = {}
    for c in counts:
        c = min(c, w.n)
        idx = order[:c]
        sub = w.subset(idx)
        wl = vt.DeviceWorkload(sub.traces, sub.slos, sub.layouts, sub.grids, [dprof], sub.scen, device=dev)
        wl.launch()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            wl.launch()
        b.record()
        b.synchronize()
        out[f"heaviest_{c}_alone_ms"] = a.elapsed_time(b) / reps
        out[f"heaviest_{c}_decisions"] = int(steps[idx].sum())
        del wl
    return out


def load_json(path):
    p = os.path.join(ROOT, path)
    return json.load(open(p)) if os.path.exists(p) else None


# ---------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2509_04827_b200 as vt
    from paper_2509_04827_b200.shard import RecordGather

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    w, parts = build_shard(args, rank, world)
    prof = w.profiles[0]
    s = fit_samples(prof)
    u32 = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).to(dev).view(torch.uint32)
    samp = dict(phase=torch.from_numpy(s["phase"]).to(dev),
                level=torch.from_numpy(s["level"].view(np.int16)).to(dev).view(torch.uint16),
                n_bt=u32(s["n_bt"]), n_req=u32(s["n_req"]), n_kv=u32(s["n_kv"]),
                lat_ms=torch.from_numpy(s["lat_ms"]).to(dev))
    n_samp = int(samp["lat_ms"].numel())
    fit = vt.fit_profile(samp["phase"], samp["level"], samp["n_bt"], samp["n_req"], samp["n_kv"], samp["lat_ms"],
                         prof.k, prof.n_tiles, prof.tile_w, 0.0)
    torch.cuda.synchronize()
    assert (fit["cell_status"].cpu().numpy() == 0).all(), "profile fit failed"
    dprof = vt.DeviceProfile.from_fit(fit, prof.mhz, prof.dyn, prof.p_idle, prof.tdp, prof.u_half_prefill,
                                      prof.u_half_decode, prof.n_tiles, prof.tile_w, dev)
    gather = RecordGather(parts, dev) if world > 1 else None
    wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, [dprof], w.scen, device=dev,
                           out=None if gather is None else gather.local)
    if gather is not None:
        gather.set_kernel_order(wl.perm)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        vt.fit_profile(samp["phase"], samp["level"], samp["n_bt"], samp["n_req"], samp["n_kv"], samp["lat_ms"],
                       prof.k, prof.n_tiles, prof.tile_w, 0.0, workspace=fit["workspace"], out=fit)
        launches = vt.last_launch_count()
        if ev:
            ev[1].record(stream)
            vt.lib().voltana_set_split_event(ev[4].cuda_event)   # recorded between K4a and K4b
        wl.launch()
        if ev:
            vt.lib().voltana_set_split_event(None)
        launches += vt.last_launch_count()
        if ev:
            ev[2].record(stream)
        if gather is not None:
            gather.enqueue()
        if ev:
            ev[3].record(stream)
        return launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    rec = wl.records()
    assert (rec["status"] == 0).all(), "scenario errors in the bench workload"
    steps_local = int((rec["steps_ctrl"] + rec["steps_route"]).sum())

    # ---------------- same-run parity gate (oracle on the fitted tables, same scenarios)
    parity, cpu = None, None
    cores = os.cpu_count() or 1
    if not args.no_parity:
        host_prof = fitted_host_profile(prof, fit)
        if world == 1 or args.scaling == "weak":
            if world == 1:
                idx, how = parity_sample(rec)
            else:   # every rank checks its own stratified sample; ranks share the host cores
                idx, how = parity_sample(rec, n_budget=ORACLE_BUDGET / world / 4)
            pool = OraclePool(dataclasses.replace(w, profiles=[host_prof]), max(1, cores // world))
            orc, wall = pool.run(idx)
            pool.close()
            parity = compare(rec[idx], orc)
            parity["sample"] = how + ("" if world == 1 else f" per rank x{world}")
            if world == 1 and not args.no_cpu_baseline:
                cpu = {"value": parity["decisions_oracle"] / wall, "unit": UNIT, "cores": pool.cores,
                       "kind": "oracle",
                       "sample": f"{how} of {args.config}, on the K1-fitted tables the GPU used (same inputs): "
                                 f"{parity['decisions_oracle']} decisions in {wall:.2f} s wall over {pool.cores} "
                                 f"processes", "decisions": parity["decisions_oracle"], "wall_s": wall}
            if world > 1:
                t = torch.tensor([parity["checked"], parity["bitexact"], int(not parity["ok"]),
                                  parity["decisions_gpu"], parity["decisions_oracle"]], dtype=torch.int64, device=dev)
                dist.all_reduce(t)
                parity.update(checked=int(t[0]), bitexact=int(t[1]), ok=int(t[2]) == 0, decisions_gpu=int(t[3]),
                              decisions_oracle=int(t[4]))
        else:   # strong: rank 0 checks the gathered sweep in global order
            gather.enqueue()
            torch.cuda.synchronize()
            allrec = gather.host_global().view(vt.RESULT_DTYPE).reshape(-1)
            ok = torch.zeros(1, dtype=torch.int64, device=dev)
            if rank == 0:
                import synth
                full = synth.build_config(args.config, seed_block=0)
                idx, how = parity_sample(allrec)
                pool = OraclePool(dataclasses.replace(full, profiles=[host_prof]), cores)
                orc, wall = pool.run(idx)
                pool.close()
                parity = compare(allrec[idx], orc)
                parity["sample"] = how + f" of the gathered sweep (strong scaling, x{world})"
                ok[0] = int(not parity["ok"])
            dist.all_reduce(ok)
            if rank != 0:
                parity = {"ok": int(ok.item()) == 0}

    # ---------------- timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(dev.index)
    clk.start()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    for e in evs:
        e[4].record(stream)   # creates the split event (torch creates events lazily)
    launches = 0
    for k in range(args.steps):
        flush.fill_(k & 0xFF)                           # L2 flush between timed steps (not timed)
        launches += step(evs[k])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    t_step = [e[0].elapsed_time(e[3]) for e in evs]
    t_fit = [e[0].elapsed_time(e[1]) for e in evs]
    t_sim = [e[1].elapsed_time(e[2]) for e in evs]
    t_pa = [e[1].elapsed_time(e[4]) for e in evs]      # setup + K4a prefill_kernel
    t_dec = [e[4].elapsed_time(e[2]) for e in evs]     # K4b simulate_kernel
    t_gather = [e[2].elapsed_time(e[3]) for e in evs]
    dev_ms = float(sum(t_step))
    tot_steps = steps_local * args.steps
    if world > 1:
        x = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        dev_ms = float(x.item())
        y = torch.tensor([tot_steps], dtype=torch.int64, device=dev)
        dist.all_reduce(y, op=dist.ReduceOp.SUM)
        tot_steps = int(y.item())
    value = tot_steps / (dev_ms / 1000.0)

    # ---------------- end to end from pinned host memory (public API), per step: H2D + kernels + D2H
    wl.pin_host()
    samp_host = {k: v.cpu().pin_memory() for k, v in samp.items()}
    h2d = d2h = 0
    e2e_ms = 0.0
    e_steps = max(1, args.e2e_steps)
    # double-buffered inputs (step k + 1's H2D overlaps step k's kernels) on one GPU; under torchrun
    # the serial path (the double-buffered one with the record all-gather has not run on a
    # multi-GPU box: gpurun gives one GPU)
    pipelined = world == 1
    if world > 1:
        dist.barrier()
    if pipelined:
        # (both buffers write their records into the same send buffer of the collective: the
        # steps are ordered on the compute stream, so one step's gather reads its own records)
        wl2 = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, [dprof], w.scen, device=dev,
                                out=None if gather is None else gather.local).pin_host()
        wls = (wl, wl2)
        samps = (samp, {k: torch.empty_like(v) for k, v in samp.items()})
        cs = torch.cuda.Stream(device=dev)
        staged = [torch.cuda.Event(), torch.cuda.Event()]
        freed = [None, None]

        def stage(x):
            if freed[x] is not None:
                cs.wait_event(freed[x])          # buffer x is free once its last step's kernels ran
            nb = wls[x].stage_inputs(stream=cs)
            with torch.cuda.stream(cs):
                for kk, v in samps[x].items():
                    v.copy_(samp_host[kk], non_blocking=True)
                    nb += v.numel() * v.element_size()
            staged[x].record(cs)
            return nb

        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        cs.wait_event(a)
        h2d = stage(0)
        for k in range(e_steps):
            x = k & 1
            flush.fill_(k & 0xFF)
            stream.wait_event(staged[x])
            sx = samps[x]
            vt.fit_profile(sx["phase"], sx["level"], sx["n_bt"], sx["n_req"], sx["n_kv"], sx["lat_ms"], prof.k,
                           prof.n_tiles, prof.tile_w, 0.0, workspace=fit["workspace"], out=fit)
            wls[x].launch()
            if gather is not None:
                gather.enqueue()
            d2h = wls[x].fetch_records()
            freed[x] = torch.cuda.Event()
            freed[x].record(stream)
            if k + 1 < e_steps:
                stage(1 - x)
        b.record(stream)
        b.synchronize()
        e2e_ms = a.elapsed_time(b)
        # both buffers produced the same records (the D2H copies are complete after b)
        assert e_steps < 2 or gather is not None or torch.equal(wl.host_out, wl2.host_out), \
            "e2e double buffers disagree"
        del wl2, samps
    else:
        for k in range(e_steps):
            flush.fill_(k & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            h2d = wl.stage_inputs()
            for kk, v in samp.items():
                v.copy_(samp_host[kk], non_blocking=True)
                h2d += v.numel() * v.element_size()
            step()
            d2h = wl.fetch_records()
            b.record(stream)
            b.synchronize()
            e2e_ms += a.elapsed_time(b)
    e2e_steps_total = steps_local * e_steps
    if world > 1:
        x = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        e2e_ms = float(x.item())
        y = torch.tensor([e2e_steps_total], dtype=torch.int64, device=dev)
        dist.all_reduce(y, op=dist.ReduceOp.SUM)
        e2e_steps_total = int(y.item())
    e2e = {"value": e2e_steps_total / (e2e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h),
           "path": "DeviceWorkload.stage_inputs (pinned H2D of traces+scenario tables+samples) -> fit_profile -> "
                   "simulate -> fetch_records (D2H)" + (
                       ", double-buffered: step k+1's H2D on a copy stream overlaps step k's kernels (and the "
                       "record all-gather when N > 1); the timed region runs from the first H2D to the last D2H"
                       if pipelined else ", serial per step")}

    # ---------------- roofline of the dominant kernel (K4b simulate_kernel)
    peaks = load_json("MEASURED_PEAKS.json") or {"hbm_gbs": 6650.0}
    fp64 = load_json("profiles/r02_fp64_peak.json")
    ncu = (load_json("profiles/ncu_traffic.json") or {}).get("simulate_kernel", {})
    K = len(w.grids[0])
    nd = w.layouts[0].n_d
    nreq = rec["n_requests"].astype(np.int64)
    pre = rec["prefill_iters"].astype(np.int64)
    dctrl = rec["steps_ctrl"].astype(np.int64) - pre
    routes = rec["steps_route"].astype(np.int64)
    k4b_s = statistics.mean(t_dec) / 1000.0
    alg_bytes = int((NODE_BYTES * nreq + RECORD_BYTES).sum())
    snap_bytes = int((32 * dctrl + (8 * nd + 16) * routes).sum())
    flops = int((dctrl * 4 * K + routes * 8 * nd * K).sum())
    achieved = alg_bytes / k4b_s / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": ncu.get("dram_bytes_per_launch"),
            "kernel": "vt::simulate_kernel (K4b: routing + decode lanes), CUDA events on the launch stream",
            "algorithmic_bytes": {"per_launch": alg_bytes,
                                  "formula": "sum over scenarios of 16 B x requests (one request node read, = the "
                                             "trace record, read once per scenario) + 128 B result record"},
            "snapshot_interface": {"per_launch": snap_bytes, "gbs": snap_bytes / k4b_s / 1e9,
                                   "frac": snap_bytes / k4b_s / 1e9 / peaks["hbm_gbs"],
                                   "formula": "32 B per decode controller decision + (8 N_D + 16) B per route "
                                              "(SURVEY 8(d))"},
            "fp64": {"ops_per_launch": flops, "achieved_gops": flops / k4b_s / 1e9,
                     "peak_gops": None if fp64 is None else fp64["fp64_gops"]["dadd"],
                     "frac": None if fp64 is None else flops / k4b_s / 1e9 / fp64["fp64_gops"]["dadd"],
                     "formula": "decode ctrl 4K + route 8 N_D K non-FMA ops per decision; peak = measured DADD "
                                "throughput (profiles/r02_fp64_peak.json)"},
            "issue": {k: ncu.get(k) for k in ("issue_pct", "occupancy_pct", "dram_gbs", "source")},
            "binding": "the latency of each scenario's serial decision chain (one warp per scenario), not HBM, "
                       "FP64 or issue throughput: see heavy-scenario times in `chain`"}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded; DESIGN.md input recipe)", "config": workload_config(args, world),
           "decisions_per_step": tot_steps // args.steps, "parity": parity,
           "kernel_ms": {"fit_profile": statistics.mean(t_fit), "simulate": statistics.mean(t_sim),
                         "simulate_prefill_k4a": statistics.mean(t_pa), "simulate_decode_k4b": statistics.mean(t_dec),
                         "all_gather": statistics.mean(t_gather) if world > 1 else 0.0},
           "fit_samples": n_samp, "gpu_launches": launches, "clocks": clocks, "e2e": e2e, "roofline": roof,
           "cpu_baseline": cpu,
           "workspace_bytes": int(wl.workspace.numel()),
           "nccl": None if world == 1 else {"backend": dist.get_backend(), "ranks": dist.get_world_size()}}
    if rank == 0:
        out["chain"] = heavy_alone(vt, torch, w, dprof, rec, dev)
        out["chain"]["strong_scaling_bound_x"] = (statistics.mean(t_sim) /
                                                  max(out["chain"]["heaviest_1_alone_ms"], 1e-9))
        if not args.no_streaming:
            out["streaming"] = streaming_kernels(vt, torch, dev, peaks["hbm_gbs"])
            out["variants"] = variant_kernels(vt, torch, w, dprof, dev)
        print(json.dumps(out), flush=True)
    ok = parity is None or parity.get("ok", True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if ok else 1


# ---------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle as it stands (test infrastructure; the tier's reference arm) on the host cores:
    each step = the oracle's K1 fit of the same 2M samples + the oracle's simulate of a bounded,
    disjoint sample of the same config's scenarios on the fitted tables."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    import synth
    w = synth.build_config(args.config, seed_block=0)
    prof = w.profiles[0]
    s = fit_samples(prof)
    cores = os.cpu_count() or 1
    per_step = min(w.n, REF_PER_STEP[args.config])
    order = np.random.default_rng(0).permutation(w.n)
    pool = OraclePool(w, cores)
    times, steps, fit_s = [], [], []
    for k in range(args.warmup + args.steps):
        idx = np.sort(order[(k * per_step) % w.n:][:per_step])
        t0 = time.perf_counter()
        f = oracle.fit_profile(s["phase"], s["level"], s["n_bt"], s["n_req"], s["n_kv"], s["lat_ms"], prof.k,
                               prof.n_tiles, prof.tile_w, 0.0)
        t1 = time.perf_counter()
        fp = dataclasses.replace(prof, **{c: f[c] for c in ("a1", "c1", "a2", "b2", "c2")})
        r, _ = pool.run(idx, fp)
        wall = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(wall)
            fit_s.append(t1 - t0)
            steps.append(int((r["steps_ctrl"] + r["steps_route"]).sum()))
    pool.close()
    value = sum(steps) / sum(times)
    sample = (f"per step: the oracle's fit of {len(s['lat_ms'])} samples (single thread, "
              f"{1000 * statistics.mean(fit_s):.0f} ms) + {per_step} random {args.config} scenarios (disjoint across "
              f"steps) on {cores} processes")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(times),
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded; DESIGN.md input recipe)", "config": workload_config(args, world),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------------- CPU dry run
def run_dry(args):
    """The multi-rank plumbing on CPU (gloo): partition, kernel-order exchange, padded record
    gather and placement in global order, max-over-ranks timing. Records are synthetic (the
    global scenario index in every byte slot), so no GPU and no oracle are involved."""
    import torch
    import torch.distributed as dist
    from paper_2509_04827_b200.shard import RecordGather
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    w, parts = build_shard(args, rank, world)
    g = RecordGather(parts, "cpu")
    mine = parts[rank]
    perm = np.random.default_rng(rank).permutation(len(mine))       # stands in for the LPT kernel order
    g.set_kernel_order(perm)
    gidx = mine[perm].astype(np.uint64)
    g.local.copy_(torch.from_numpy(np.repeat(gidx, 16).view(np.uint8).reshape(len(mine), 128)))
    t0 = time.perf_counter()
    g.enqueue()
    ms = (time.perf_counter() - t0) * 1000
    x = torch.tensor([ms], dtype=torch.float64)
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    res = g.host_global()
    ok = bool((res.view(np.uint64)[:, 0] == np.arange(g.n_total, dtype=np.uint64)).all())
    if rank == 0:
        print(json.dumps({"dry_run": True, "backend": dist.get_backend(), "ranks": dist.get_world_size(),
                          "scaling": args.scaling, "config": args.config, "n_total": g.n_total,
                          "parts": [len(p) for p in parts], "gather_ok": ok, "gather_ms_max": float(x.item())}),
              flush=True)
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a))
    if a.impl == "reference":
        sys.exit(run_reference(a))
    if a.dry_run:
        sys.exit(run_dry(a))
    sys.exit(run_ours(a))
