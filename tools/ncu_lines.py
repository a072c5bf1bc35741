"""Per-CUDA-source-line totals (stall samples, instructions) from
`ncu --page source --csv --print-source cuda,sass`; multiple files supported."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
cur_file, hdr = None, None
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
line = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0].strip():
        line = (cur_file, int(r[0])); agg[line][2] = r[1][:90]
    if line is None: continue
    try:
        agg[line][0] += float(r[4] or 0); agg[line][1] += float(r[7] or 0)
    except ValueError:
        pass
tot_s = sum(v[0] for v in agg.values()); tot_i = sum(v[1] for v in agg.values())
print(f"total samples {tot_s:.0f}, instructions {tot_i:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{k[0]:>16s}:{k[1]:<4d} {100*v[0]/tot_s:5.1f}% st {100*v[1]/tot_i:5.1f}% in | {v[2]}")
