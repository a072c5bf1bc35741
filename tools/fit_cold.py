"""K1 fit of the bench's 2 M recording-order samples: CUDA-event time back to back (warm L2)
vs after a 256 MiB L2-flush write each call (as in bench.py's step)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, bench, paper_2509_04827_b200 as vt
prof = synth.make_profile("L8")
s = bench.fit_samples(prof)
u32 = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda().view(torch.uint32)
d = dict(phase=torch.from_numpy(s["phase"]).cuda(), level=torch.from_numpy(s["level"].view(np.int16)).cuda().view(torch.uint16),
         n_bt=u32(s["n_bt"]), n_req=u32(s["n_req"]), n_kv=u32(s["n_kv"]), lat_ms=torch.from_numpy(s["lat_ms"]).cuda())
f = lambda **kw: vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, prof.n_tiles, prof.tile_w, 0.0, **kw)
fo = f()
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
for mode in ("warm", "flushed", "flushed+sync"):
    ts = []
    for r in range(12):
        if mode != "warm":
            flush.fill_(r & 0xff)
        if mode == "flushed+sync":
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(workspace=fo["workspace"], out=fo); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    print(mode, "ms per call (median of 12):", round(float(np.median(ts[2:])), 4), flush=True)
for nrep in (1, 2, 5, 10, 20):
    ts = []
    for r in range(6):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(nrep):
            f(workspace=fo["workspace"], out=fo)
        b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{nrep} back-to-back calls: {float(np.median(ts[1:])):.4f} ms", flush=True)
# host-side cost of one call (no GPU wait)
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    f(workspace=fo["workspace"], out=fo)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host time per call: {(t1 - t0) / 20 * 1e3:.4f} ms", flush=True)
