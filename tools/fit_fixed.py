"""K1 fixed cost: CUDA-event time of fit_profile at a few sample counts (recording order)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2509_04827_b200 as vt
from synth.samples import profile_samples
prof = synth.make_profile("L8")
for per_cell in (8, 64, 512, 4096, 32768):
    smp = profile_samples(prof, per_cell, per_cell, noise_sigma=0.02, seed=9, shuffle=False)
    to = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else (a.view(np.int16) if a.dtype == np.uint16 else a)).cuda()
    d = {k: to(v) for k, v in smp.items()}
    for k in ("n_bt", "n_req", "n_kv"):
        d[k] = d[k].view(torch.uint32)
    d["level"] = d["level"].view(torch.uint16)
    f = lambda **kw: vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, prof.n_tiles, **kw)
    fo = f()
    for _ in range(10):
        f(workspace=fo["workspace"], out=fo)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        f(workspace=fo["workspace"], out=fo)
    b.record(); b.synchronize()
    n = int(d["lat_ms"].numel())
    print(f"n={n:9d}  {a.elapsed_time(b) / 50 * 1e3:8.1f} us", flush=True)
