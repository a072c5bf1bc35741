"""SASS instructions (with executed counts and stall samples) that the line table maps to given
source lines. Usage: python tools/ncu_line_sass.py REPORT KERNEL OBJ FILE:LINE [FILE:LINE ...]"""
import csv, io, os, re, subprocess, sys, tempfile
rep, kern, obj = sys.argv[1], sys.argv[2], sys.argv[3]
want = set(sys.argv[4:])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + kern.split("ILi")[0].replace("_ZN2vt", "").lstrip("0123456789")],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
col = {n: i for i, n in enumerate(rows[h])}
data = [r for r in rows[h + 1:] if r and r[0].startswith("0x")]
base = int(data[0][0], 16)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):
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
for r in data:
    off = int(r[0], 16) - base
    if line_of.get(off) in want:
        print(f"{line_of[off]:20s} {off:6x} {r[col['Instructions Executed']]:>8s} {r[col['Warp Stall Sampling (All Samples)']]:>6s}  {r[col['Source']].strip()[:70]}")
