"""One K1 fit of synthetic samples under a wall clock (hang / latency check).

    python tools/fit_dbg.py L8|B200 N_TILES PER_CELL SHUFFLE(0|1)
"""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth, paper_2509_04827_b200 as vt
from synth.samples import profile_samples
kind, T, ncell, shuf = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] == "1"
prof = synth.make_profile(kind, n_tiles=T)
s = profile_samples(prof, ncell * 2, ncell, noise_sigma=0.05, seed=11, shuffle=shuf)
d = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int32) if v.dtype == np.uint32 else v).to("cuda") for k, v in s.items()}
for k in ("n_bt", "n_req", "n_kv"):
    d[k] = d[k].view(torch.uint32)
d["level"] = torch.from_numpy(s["level"].view(np.int16)).to("cuda").view(torch.uint16)
print("n", len(s["lat_ms"]), flush=True)
t = time.time()
out = vt.fit_profile(d["phase"], d["level"], d["n_bt"], d["n_req"], d["n_kv"], d["lat_ms"], prof.k, T, 128, 1.5)
print("launched", flush=True)
torch.cuda.synchronize()
print("done", time.time() - t, out["cell_status"].cpu().numpy()[:10], flush=True)
