"""Sum ncu gpu__time_duration per kernel name over the LAST step of each launch list; print side by side."""
import csv
import sys
from collections import OrderedDict


def load(p):
    rows = []
    with open(p) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"].split("(")[0][:60], float(r["Metric Value"].replace(",", "")),
                         r.get("Metric Unit", "")))
    return rows


def last_step(rows):
    # the step starts at the first pack kernel after warmup: take everything from the last 'pack' occurrence
    idx = [i for i, r in enumerate(rows) if "pack_meta" in r[0] or "pack_offsets" in r[0]]
    start = idx[-1] if idx else 0
    return rows[start:]


tabs = []
for p in sys.argv[1:]:
    rows = last_step(load(p))
    d = OrderedDict()
    for n, v, u in rows:
        v = v / 1000.0 if u in ("nsecond", "ns") else v
        d[n] = d.get(n, 0.0) + v
    tabs.append(d)
names = list(OrderedDict.fromkeys(n for t in tabs for n in t))
print("kernel".ljust(62), *[f"{i:>10}" for i in range(len(tabs))])
for n in names:
    print(n.ljust(62), *[f"{t.get(n, 0.0):10.1f}" for t in tabs])
print("TOTAL (us)".ljust(62), *[f"{sum(t.values()):10.1f}" for t in tabs])
