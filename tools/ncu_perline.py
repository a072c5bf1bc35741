"""Instructions executed and stall samples per CUDA source line (ncu source page + the cubin's
line table). Usage: python tools/ncu_perline.py REPORT KERNEL OBJ UNITS [lo-hi] [top]"""
import csv, io, os, re, subprocess, sys, tempfile
from collections import defaultdict
rep, kern, obj, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
lo, hi = (map(int, sys.argv[5].split("-")) if len(sys.argv) > 5 else (0, 10**9))
top = int(sys.argv[6]) if len(sys.argv) > 6 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern.split("ILi")[0].replace("_ZN2vt", "").lstrip("0123456789")],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
H = rows[h]; col = {n: i for i, n in enumerate(H)}
data = [r for r in rows[h + 1:] if r and r[0].startswith("0x")]
base = int(data[0][0], 16)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):   # the cubin holding the kernel
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout.splitlines()
    st = next((i for i, l in enumerate(dis) if l.startswith("//--------------------- .text." + kern)), None)
    if st is not None:
        break
line_of, cur = {}, "?"
for l in dis[st + 1:]:
    if l.startswith("//--------------------- .text."):
        break
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"; continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
inst, samp = defaultdict(float), defaultdict(float)
for r in data:
    ln = line_of.get(int(r[0], 16) - base, "?")
    inst[ln] += float(r[col["Instructions Executed"]] or 0)
    samp[ln] += float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
T = sum(samp.values())
src = {}
for f in ("k_simulate.cu", "k_decide.cu", "k_fit.cu"):
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2509_04827_b200", "csrc", f)
    src[f] = open(p).read().splitlines()
sel = [(k, v) for k, v in inst.items() if k.split(":")[0] in src and lo <= int(k.split(":")[1]) <= hi]
if os.environ.get("OTHER"):
    for k in sorted(samp, key=lambda k: -samp[k])[:12]:
        print(f"{100*samp[k]/T:5.1f}% {inst[k]/units:7.2f}/u  {k}")
    sys.exit(0)
for k, v in sorted(sel, key=lambda kv: -(samp[kv[0]] if os.environ.get("BY_STALL") else kv[1]))[:top]:
    f, n = k.split(":")
    print(f"{v / units:7.1f}/u {100 * samp[k] / T:5.1f}%  {k:20s} {src[f][int(n) - 1].strip()[:90]}")
