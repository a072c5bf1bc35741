"""Per-scenario features and measured K4 durations (debug timing hook) -> npz, for fitting
the host-side LPT cost model of DeviceWorkload.

    python tools/scen_dump.py [--config C4] [--out gpurun_out/scen_C4.npz]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2509_04827_b200 as vt

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4"); ap.add_argument("--out", default=None)
a = ap.parse_args()
w = synth.build_config(a.config)
wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
wl.launch(); torch.cuda.synchronize()
buf = torch.zeros(2 * wl.n, dtype=torch.int64, device="cuda")
vt.lib().voltana_debug_set_timing(buf.data_ptr())
wl.launch(); torch.cuda.synchronize()
vt.lib().voltana_debug_set_timing(None)
tm = buf.cpu().numpy().view(np.uint64).reshape(-1, 2)
t0 = tm[:, 0].astype(np.int64)
dur = (tm[:, 1] & np.uint64((1 << 56) - 1)).astype(np.int64)
rec = wl.out.cpu().numpy().view(vt.RESULT_DTYPE).reshape(-1)     # kernel (LPT) order
inv = wl.inv
off = np.asarray(w.traces.offset, np.int64)
tid = np.asarray(w.scen["trace_id"], np.int64)
N = np.diff(off)[tid]
cs_in = np.concatenate([[0], np.cumsum(np.asarray(w.traces.in_len, np.int64))])
cs_out = np.concatenate([[0], np.cumsum(np.asarray(w.traces.out_len, np.int64))])
sum_in = (cs_in[off[1:]] - cs_in[off[:-1]])[tid]
sum_out = (cs_out[off[1:]] - cs_out[off[:-1]])[tid]
slo = np.asarray(w.scen["slo_id"], np.int64)
lay = np.asarray(w.scen["layout_id"], np.int64)
np.savez(a.out or f"gpurun_out/scen_{a.config}.npz",
         N=N, sum_in=sum_in, sum_out=sum_out, duration=np.asarray(w.traces.duration)[tid],
         slo_itl=np.array([w.slos[i].itl for i in slo]), slo_ttft=np.array([w.slos[i].ttft for i in slo]),
         n_d=np.array([w.layouts[i].n_d for i in lay]), n_p=np.array([w.layouts[i].n_p for i in lay]),
         steps_ctrl=rec["steps_ctrl"][inv], steps_route=rec["steps_route"][inv],
         gpu_ns=dur[inv], start_ns=(t0 - t0.min())[inv], perm=wl.perm)
print("ok", wl.n, "span ms", ((t0 + dur).max() - t0.min()) / 1e6)
