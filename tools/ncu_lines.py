"""Aggregate an ncu source page (SASS, stall samples) by CUDA source line, using the line
table of the build's cubin (nvdisasm -g). Usage:
    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_MANGLED OBJ.o [top]
"""
import csv
import io
import re
import subprocess
import sys
import tempfile
import os
from collections import defaultdict

rep, kern, obj = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern.split("ILi")[0].replace("_ZN2vt", "").lstrip("0123456789")],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
H = rows[hdr]
col = {n: i for i, n in enumerate(H)}
data = [r for r in rows[hdr + 1:] if r and r[0].startswith("0x")]
base = int(data[0][0], 16)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith("//--------------------- .text." + kern))
line_of = {}
cur = "?"
for l in dis[start + 1:]:
    if l.startswith("//--------------------- .text."):
        break
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
stalls = [n for n in H if n.startswith("stall_") and "Not Issued" not in n]
agg = defaultdict(lambda: defaultdict(float))
tot = 0.0
for r in data:
    off = int(r[0], 16) - base
    ln = line_of.get(off, "?")
    s = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    agg[ln]["samples"] += s
    agg[ln]["inst"] += float(r[col["Instructions Executed"]] or 0)
    for n in stalls:
        agg[ln][n] += float(r[col[n]] or 0)
    tot += s
print(f"total samples {tot:.0f}")
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    top3 = sorted(((v[n], n[6:]) for n in stalls), reverse=True)[:3]
    print(f"{100 * v['samples'] / tot:5.1f}%  {ln:28s} inst {v['inst']:>10.0f}  " +
          ", ".join(f"{k} {100 * x / max(v['samples'], 1):.0f}%" for x, k in top3 if x > 0))

# ---- regions (k_simulate.cu line ranges given as extra args "name:lo-hi")
regions = [a for a in sys.argv[5:] if ":" in a]
if regions:
    print("--- regions")
    for reg in regions:
        name, rng = reg.split(":")
        lo, hi = map(int, rng.split("-"))
        s = i = 0.0
        for ln, v in agg.items():
            if ln.startswith("k_simulate.cu:") and lo <= int(ln.split(":")[1]) <= hi:
                s += v["samples"]
                i += v["inst"]
        print(f"{name:16s} samples {100 * s / tot:5.1f}%  inst {i:>12.0f}")
    other = sum(v["inst"] for ln, v in agg.items() if not ln.startswith("k_simulate.cu:"))
    print(f"{'non-k_simulate':16s} inst {other:>12.0f}")
