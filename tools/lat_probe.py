"""Per-phase clock64 cycles of K4b's route loop (build with -DVT_LAT_PROBE; VOLTANA_SO=that build):
select + stream advance / decode advance / EcoRoute + push / drain + ITL pass, per route.

    VOLTANA_SO=variants/lib_lat.so python tools/lat_probe.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2509_04827_b200 as vt

for name, idx in (("148 heaviest alone", np.array([s * 1024 + 896 + q for s in range(4) for q in range(37)])),
                  ("full C4", None)):
    w = synth.build_config("C4", scenarios=idx)
    wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
    wl.launch(); torch.cuda.synchronize()
    buf = torch.zeros(6 * wl.n, dtype=torch.int64, device="cuda")
    vt.lib().voltana_debug_set_timing(buf.data_ptr())
    wl.launch(); torch.cuda.synchronize()
    vt.lib().voltana_debug_set_timing(None)
    t = buf.cpu().numpy().view(np.uint64)[2 * wl.n:].reshape(-1, 4).astype(np.float64)
    rec = wl.out.cpu().numpy().view(vt.RESULT_DTYPE).reshape(-1)
    routes = rec["steps_route"].astype(np.float64)
    dec = (rec["steps_ctrl"] - rec["prefill_iters"]).astype(np.float64)
    tot = t.sum(axis=1)
    k = np.argsort(-tot)[:16]   # the longest scenarios
    per = t[k].sum(axis=0) / routes[k].sum()
    print(f"{name}: longest 16 scenarios, cycles per route: select+advance-stream {per[0]:.0f}, "
          f"decode advance {per[1]:.0f} ({dec[k].sum() / routes[k].sum():.2f} decode iterations per route), "
          f"EcoRoute+push {per[2]:.0f}, drain+ITL pass {per[3]:.0f}; total {per.sum():.0f} cycles/route "
          f"= {per.sum() / 1.965:.0f} ns at 1965 MHz", flush=True)
