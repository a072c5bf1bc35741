"""One warm call each of K2 control_step (2^25 snapshots), K3 route_batch (2^24 items) and K1
fit_profile (32768 samples per cell of the L8 profile, 15.6 M samples) — for ncu captures.

    ncu --set full -k regex:"control_kernel|route_kernel|fit_kernel" -c 4 python tools/prof_stream.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from synth.samples import profile_samples
import paper_2509_04827_b200 as vt

dev = torch.device("cuda")
prof = synth.make_profile("L8")
dp = vt.DeviceProfile(prof, dev)
lad = [0, 6, 13, 20, 27]
g = torch.Generator(device=dev).manual_seed(0)
u32 = lambda lo, hi, size: torch.randint(lo, hi, size, generator=g, device=dev, dtype=torch.int64).to(torch.int32).view(torch.uint32)
n = 1 << 25
load, kv = u32(1, 700, (n,)), u32(700, 300000, (n,))
q = (torch.rand(n, generator=g, device=dev) < 0.05).to(torch.int32).view(torch.uint32)
tgt = torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 60 + 20
m = 1 << 24
nr, nk, rin = u32(0, 500, (2 * m,)), u32(500, 200000, (2 * m,)), u32(1, 4000, (m,))
cur = torch.zeros(m, dtype=torch.int32, device=dev).view(torch.uint32)
smp = profile_samples(prof, 32768, 32768, noise_sigma=0.02, seed=9, shuffle=False)
to = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else (a.view(np.int16) if a.dtype == np.uint16 else a)).to(dev)
d = {k: to(v) for k, v in smp.items()}
for k in ("n_bt", "n_req", "n_kv"):
    d[k] = d[k].view(torch.uint32)
d["level"] = d["level"].view(torch.uint16)
for rep in range(2):   # launch order per rep: control, route, fit (one cooperative launch)
    vt.control_step(dp, 1, lad, load, kv, q, None, tgt)
    vt.route_batch(dp, lad, 2, nr, nk, rin, tgt[:m], 150, 0, cur)
    fo = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, prof.n_tiles)
torch.cuda.synchronize()
print("ok", int(d["lat_ms"].numel()))
