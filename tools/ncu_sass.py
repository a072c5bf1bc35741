"""Summarise an ncu --page source --print-source sass CSV: stall totals and hottest instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]] or 0)
    except (ValueError, KeyError): return 0.0
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in data:
    for s in stalls: tot[s] += f(r, s)
S = sum(tot.values())
print("stall breakdown (% of samples):")
for s, v in tot.most_common(12): print(f"  {s:28s} {100*v/S:5.1f}")
ins = sum(f(r, "Instructions Executed") for r in data)
print(f"instructions executed: {ins:.3e}")
top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    print(f'{r[ix["Address"]]:>8s} {f(r,"Warp Stall Sampling (All Samples)"):8.0f} {f(r,"Instructions Executed"):10.0f}  {r[ix["Source"]][:70]}')
