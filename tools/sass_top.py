"""Hottest SASS instructions of one kernel section of an `ncu --page source --csv --print-source sass` export.
Usage: python tools/sass_top.py CSV [section index] [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]; secs.append(cur)
    elif r and r[0] == "Address":
        cur[1] = {h: i for i, h in enumerate(r)}
    elif r and r[0].startswith("0x") and cur is not None:
        cur[2].append(r)
name, ix, data = secs[int(sys.argv[2]) if len(sys.argv) > 2 else 0]
S = lambda r: float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
I = lambda r: float(r[ix["Instructions Executed"]] or 0)
tot = sum(S(r) for r in data)
print(name, "samples", tot, "instructions", sum(I(r) for r in data))
top = sorted(range(len(data)), key=lambda i: -S(data[i]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]
for i in sorted(top):
    r = data[i]
    print(f"{i:5d} {100 * S(r) / tot:5.1f}% {int(I(r)):10d}  {r[ix['Source']][:70]}")
