"""Simulate a chosen subset of a config (default: the single heaviest C4 scenario) — for ncu
source-level captures of K4b's serial chain and for latency experiments.

    python tools/prof_one.py [--config C4] [--heaviest 1] [--reps 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_2509_04827_b200 as vt

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--heaviest", type=int, default=1, help="the k scenarios with the longest traces")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--index", type=int, nargs="*", default=None, help="explicit scenario indices instead of --heaviest")
a = ap.parse_args()
w = synth.build_config(a.config)
lens = w.traces.lengths()[w.scen["trace_id"]].astype(np.int64)
# heaviest = longest trace, most demanding SLO first (stable on scenario index)
idx = np.argsort(-lens, kind="stable")[:a.heaviest] if a.index is None else np.array(a.index)
sub = w.subset(idx)
wl = vt.DeviceWorkload(sub.traces, sub.slos, sub.layouts, sub.grids, sub.profiles, sub.scen)
for r in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    wl.launch()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
rec = wl.records()
st = int((rec["steps_ctrl"] + rec["steps_route"]).sum())
print(f"{a.config} heaviest {len(idx)}: {dt * 1e3:.2f} ms wall, {st} decisions, "
      f"{int(rec['steps_route'].sum())} routes", flush=True)
