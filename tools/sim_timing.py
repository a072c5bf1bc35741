"""Per-scenario timeline of voltana_simulate (debug timing hook): tail vs throughput.

    python tools/sim_timing.py [--config C4] [--n 0] [--scale 1.0]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2509_04827_b200 as vt

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4"); ap.add_argument("--n", type=int, default=0)
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
full = {"C1": 1, "C2": 1024, "C3": 256, "C4": 4096, "C5": 16384}[a.config]
idx = None if a.n == 0 else np.linspace(0, full - 1, a.n).astype(int)
w = synth.build_config(a.config, scenarios=idx, duration_scale=a.scale)
wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
wl.launch(); torch.cuda.synchronize()
buf = torch.zeros(2 * wl.n, dtype=torch.int64, device="cuda")
vt.lib().voltana_debug_set_timing(buf.data_ptr())
wl.launch(); torch.cuda.synchronize()
vt.lib().voltana_debug_set_timing(None)
tm = buf.cpu().numpy().view(np.uint64).reshape(-1, 2)
t0 = tm[:, 0].astype(np.int64); t1 = t0 + (tm[:, 1] & np.uint64((1 << 56) - 1)).astype(np.int64)
sm = (tm[:, 1] >> 56).astype(np.int64)
rec = wl.out.cpu().numpy().view(vt.RESULT_DTYPE).reshape(-1)     # LPT (launch) order
steps = (rec["steps_ctrl"] + rec["steps_route"]).astype(np.int64)
base = t0.min(); span = (t1.max() - base) / 1e6
dur = (t1 - t0) / 1e6
print(f"span {span:.2f} ms, scenarios {wl.n}, decisions {steps.sum()}, {steps.sum()/span/1e6:.1f} G steps/s")
print(f"scenario ms: min {dur.min():.2f} median {np.median(dur):.2f} max {dur.max():.2f}; "
      f"ns/decision median {np.median(dur*1e6/np.maximum(steps,1)):.0f} (max-scenario {dur.max()*1e6/steps[np.argmax(dur)]:.0f})")
ts = np.linspace(0, span, 41)
conc = [int(((t0 - base) / 1e6 <= x).sum() - ((t1 - base) / 1e6 <= x).sum()) for x in ts]
print("concurrency over time:", conc)
print("start offsets (ms) of last 10 claimed:", np.round((np.sort(t0)[-10:] - base) / 1e6, 2))
last = np.argsort(t1)[-5:]
print("last finishers: dur ms", np.round(dur[last], 2), "steps", steps[last], "start", np.round((t0[last]-base)/1e6, 2))
print("per-SM busy spread (ms):", np.round(np.percentile([dur[sm == s].sum() for s in np.unique(sm)], [0, 50, 100]), 1))
