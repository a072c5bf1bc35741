"""K4a per-chain timeline (build with -DVT_PA_TIMING; VOLTANA_SO=that build).

    VOLTANA_SO=variants/lib_patime.so python tools/pa_timing.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2509_04827_b200 as vt

w = synth.build_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
wl.launch(); torch.cuda.synchronize()
npm = max(x.n_p for x in w.layouts)
buf = torch.zeros(2 * wl.n + 2 * wl.n * npm, dtype=torch.int64, device="cuda")
vt.lib().voltana_debug_set_timing(buf.data_ptr())
wl.launch(); torch.cuda.synchronize()
vt.lib().voltana_debug_set_timing(None)
tm = buf.cpu().numpy().view(np.uint64)[2 * wl.n:].reshape(-1, 2).astype(np.int64)
t0 = tm[:, 0]; du = tm[:, 1]
ok = t0 > 0
t0 = t0[ok]; du = du[ok]
base = t0.min(); t1 = t0 + du
span = (t1.max() - base) / 1e6
rec = wl.out.cpu().numpy().view(vt.RESULT_DTYPE).reshape(-1)
pit = np.repeat(rec["prefill_iters"].astype(np.int64) / npm, npm)[ok]
print(f"K4a span {span:.2f} ms, chains {ok.sum()}; chain ms: median {np.median(du)/1e6:.2f} max {du.max()/1e6:.2f}")
print(f"ns per batch (chain dur / batches): median {np.median(du/np.maximum(pit,1)):.0f}, for the longest chain "
      f"{du[np.argmax(du)]/max(pit[np.argmax(du)],1):.0f} ({pit[np.argmax(du)]:.0f} batches)")
ts = np.linspace(0, span, 21)
print("concurrency:", [int(((t0 - base) / 1e6 <= x).sum() - ((t1 - base) / 1e6 <= x).sum()) for x in ts])
print("start of last 5 chains (ms):", np.round((np.sort(t0)[-5:] - base) / 1e6, 2))
