"""Top SASS instructions by warp-stall samples from `ncu --page source --csv` (per-instruction stall reasons)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) == len(hdr)]
tot = Counter()
for r in data:
    for h in reasons:
        try:
            tot[h] += int(r[ix[h]])
        except ValueError:
            pass
allsamp = sum(int(r[2]) for r in data if r[2].isdigit())
print("total samples", allsamp)
for h, v in tot.most_common(12):
    print(f"  {h:28s} {v:8d} {100.0 * v / max(allsamp, 1):5.1f}%")
top = sorted(data, key=lambda r: -int(r[2]) if r[2].isdigit() else 0)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for r in top:
    rs = sorted(((int(r[ix[h]]) if r[ix[h]].isdigit() else 0, h) for h in reasons), reverse=True)[:3]
    print(f"{r[0][-5:]} {int(r[2]):6d}  {r[1].strip()[:60]:60s} " + " ".join(f"{h[6:]}={v}" for v, h in rs if v))
