"""Time only the heaviest C4 scenarios (lambda = 75: 512 of 4096) with the GPU otherwise idle:
their per-decision latency without co-resident warps vs inside the full sweep."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2509_04827_b200 as vt

for name, idx in (("lambda=75 x 512", np.array([s * 1024 + 896 + q for s in range(4) for q in range(128)])),
                  ("lambda=75 x 148", np.array([s * 1024 + 896 + q for s in range(4) for q in range(37)]))):
    w = synth.build_config("C4", scenarios=idx)
    wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
    for r in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter(); wl.launch(); torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    rec = wl.records()
    st = int((rec["steps_ctrl"] + rec["steps_route"]).sum())
    print(f"{name}: {dt*1e3:.1f} ms, {st} decisions, max per scenario {int((rec['steps_ctrl'] + rec['steps_route']).max())}", flush=True)
