"""The 148 heaviest C4 scenarios alone (one warp per SM): for a source-level ncu capture of
the single-scenario critical path (no co-resident warps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2509_04827_b200 as vt
idx = np.array([s * 1024 + 896 + q for s in range(4) for q in range(37)])
w = synth.build_config("C4", scenarios=idx)
wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
wl.launch(); torch.cuda.synchronize()
print("ok")
