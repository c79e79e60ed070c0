#!/usr/bin/env python
"""DRAM traffic per kernel class from an ncu metrics CSV (scripts/gpu_traffic.sh):
dram__bytes_read.sum + dram__bytes_write.sum summed over the LAST bench step's launches.
Usage: python scripts/traffic_summary.py gpurun_out/TAG_traffic.csv > profiles/rNN_dram_traffic.json"""
import collections
import csv
import json
import sys


def klass(name: str) -> str:
    if "gemm" in name:
        return "gemm"
    if "attn_fwd_kernel" in name:
        return "attn_fwd"
    if "attn_bwd_dq_kernel" in name or "attn_bwd_dkv_kernel" in name or "attn_bwd_dq2_kernel" in name:
        return "attn_bwd"
    return "other"


rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
per = collections.OrderedDict()
for d in data:
    per.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"])
launches = list(per.values())
# the last step starts at the pack_offsets launch right before the last pack_rows launch (the
# row-move pack, issued first by CadetStack.step on its side stream)
start = max(i for i, l in enumerate(launches) if "pack_rows" in l["name"]) - 1
step = launches[start:]
agg = collections.defaultdict(lambda: {"dram_bytes_per_step": 0.0, "launches": 0, "time_us": 0.0})
for l in step:
    a = agg[klass(l["name"])]
    a["dram_bytes_per_step"] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
    a["launches"] += 1
    a["time_us"] += l.get("gpu__time_duration.sum", 0.0) / 1e3
for a in agg.values():
    a["dram_bytes_per_launch"] = a["dram_bytes_per_step"] / a["launches"]
out = {"source": sys.argv[1].split("/")[-1],
       "method": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 "--clock-control none, last step of bench.py --steps 2 --warmup 1",
       **agg}
print(json.dumps(out, indent=1))
