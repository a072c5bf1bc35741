"""Per-kernel launch counts, mean duration and share of GPU time from an ncu
`--metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_share.py gpurun_out/launches.csv "<command>" > profiles/rNN_launches_share.json
"""
import csv, json, sys, collections
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[ui], 1.0)
    agg[r[ki].split("(")[0]].append(v)
tot = sum(sum(v) for v in agg.values())
out = {"command": sys.argv[2] if len(sys.argv) > 2 else "",
       "kernels": {k: {"launches": len(v), "mean_ms": sum(v) / len(v), "share_of_gpu_time": sum(v) / tot}
                   for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}}
print(json.dumps(out, indent=1))
