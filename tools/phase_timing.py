"""Phase-A share of each scenario's time (build with -DVT_PHASE_TIMING; VOLTANA_SO=that build).

    VOLTANA_SO=variants/lib_phase.so python tools/phase_timing.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2509_04827_b200 as vt

w = synth.build_config("C4")
wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
wl.launch(); torch.cuda.synchronize()
buf = torch.zeros(2 * wl.n, dtype=torch.int64, device="cuda")
vt.lib().voltana_debug_set_timing(buf.data_ptr())
wl.launch(); torch.cuda.synchronize()
vt.lib().voltana_debug_set_timing(None)
tm = buf.cpu().numpy().view(np.uint64).reshape(-1, 2)
pa = tm[:, 0].astype(np.float64) / 1e6
tot = (tm[:, 1] & np.uint64((1 << 56) - 1)).astype(np.float64) / 1e6
print(f"phase A: total {pa.sum():.0f} warp-ms of {tot.sum():.0f} ({100 * pa.sum() / tot.sum():.1f} %); "
      f"per scenario median {np.median(pa):.2f} ms of {np.median(tot):.2f} ms")
