"""Launch voltana_simulate on a (reduced) config for ncu / timing experiments.

    python tools/prof_sim.py [--config C4] [--n 512] [--scale 0.25] [--reps 2]
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
ap.add_argument("--n", type=int, default=0, help="scenarios (0 = all)")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
full = {"C1": 1, "C2": 1024, "C3": 256, "C4": 4096, "C5": 16384}[a.config]
idx = None if a.n == 0 else np.linspace(0, full - 1, a.n).astype(int)
w = synth.build_config(a.config, scenarios=idx, duration_scale=a.scale)
wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
for r in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    wl.launch()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rec = wl.records()
    steps = int((rec["steps_ctrl"] + rec["steps_route"]).sum())
    print(f"rep {r}: {w.n} scenarios, {steps} decisions, {dt*1e3:.2f} ms, {steps/dt/1e6:.1f} M steps/s", flush=True)
