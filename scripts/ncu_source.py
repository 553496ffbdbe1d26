"""Top stall locations of an ncu --page source --csv export (SASS level)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
I = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[I["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
agg = {s: sum(int(r[I[s]] or 0) for r in data) for s in stalls}
for s, v in sorted(agg.items(), key=lambda x: -x[1])[:8]:
    print(f"  {s:24s} {v:7d} {v / max(tot, 1):6.1%}")
top = sorted(data, key=lambda r: -int(r[I["Warp Stall Sampling (All Samples)"]] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    n = int(r[I["Warp Stall Sampling (All Samples)"]] or 0)
    main = max(stalls, key=lambda s: int(r[I[s]] or 0))
    print(f"{n:6d} {n / max(tot, 1):5.1%} {main:18s} {r[I['Address']][-5:]} {r[I['Source']].strip()[:70]}")
