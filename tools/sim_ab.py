"""A/B timing of K4 builds on one config: for each .so given, the K4b (simulate_kernel) time
of voltana_simulate over the full sweep (CUDA events around K4b via the split event), the
whole call, and the records' hash (must be equal across builds).

    python tools/sim_ab.py [--config C4] [--reps 5] lib1.so lib2.so ...   (each in a subprocess)
"""
import argparse
import json
import os
import subprocess
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--child", default=None)
ap.add_argument("libs", nargs="*")
a = ap.parse_args()
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if a.child is None:
    for so in a.libs:
        env = dict(os.environ, VOLTANA_SO=os.path.abspath(so))
        r = subprocess.run([sys.executable, __file__, "--config", a.config, "--reps", str(a.reps), "--child", so],
                           env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)
    sys.exit(0)

sys.path.insert(0, ROOT)
import hashlib
import numpy as np
import torch
import synth
import paper_2509_04827_b200 as vt

w = synth.build_config(a.config)
wl = vt.DeviceWorkload(w.traces, w.slos, w.layouts, w.grids, w.profiles, w.scen)
wl.launch()
torch.cuda.synchronize()
k4b, call = [], []
for _ in range(a.reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[1].record()
    e[0].record()
    vt.lib().voltana_set_split_event(e[1].cuda_event)
    wl.launch()
    vt.lib().voltana_set_split_event(None)
    e[2].record()
    torch.cuda.synchronize()
    k4b.append(e[1].elapsed_time(e[2]))
    call.append(e[0].elapsed_time(e[2]))
rec = wl.records()
h = hashlib.sha1(rec.tobytes()).hexdigest()[:12]
print(json.dumps({"lib": a.child, "k4b_ms": round(float(np.median(k4b)), 2), "k4b_min": round(min(k4b), 2),
                  "call_ms": round(float(np.median(call)), 2), "records_sha1": h}))
