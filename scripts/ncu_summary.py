#!/usr/bin/env python
"""Summarise ncu evidence into profiles/: per-kernel share from a launch list (gpu__time_duration)
and key metrics from `ncu --set full` reports.  Usage:
  python scripts/ncu_summary.py TAG [launches.csv] [rep1.ncu-rep ...] > profiles/TAG_ncu_summary.md"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "TMEM active % (tcgen05)"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "smem pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    return [d for d in data if d.get("Metric Name") == "gpu__time_duration.sum"]


def main():
    tag = sys.argv[1]
    print(f"# ncu summary {tag}\n")
    for a in sys.argv[2:]:
        if a.endswith(".csv"):
            data = launch_list(a)
            # a step starts at the pack_offsets launch right before its row-move pack (pack_rows)
            starts = [i - 1 for i, d in enumerate(data) if "pack_rows_kernel" in d["Kernel Name"]]
            step = data[starts[-1]:] if starts else data
            tot = sum(float(d["Metric Value"]) for d in step)
            agg = collections.OrderedDict()
            for d in step:
                k = d["Kernel Name"].split("(")[0].replace("void ", "")
                agg.setdefault(k, [0.0, 0])
                agg[k][0] += float(d["Metric Value"])
                agg[k][1] += 1
            print(f"## Launch list `{a.split('/')[-1]}` - last step: {len(step)} launches, {tot/1e3:.1f} us "
                  f"(cold-cache, serialised by ncu: compare shares, not absolutes)\n")
            print("| kernel | launches | time (us) | share |\n|---|---|---|---|")
            for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
                print(f"| {k} | {n} | {t/1e3:.1f} | {100*t/tot:.1f}% |")
            print()
        elif a.endswith(".ncu-rep"):
            out = subprocess.run(["ncu", "-i", a, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
            rows = list(csv.reader(io.StringIO(out)))
            if len(rows) < 3:
                continue
            hdr, units = rows[0], rows[1]
            print(f"## `{a.split('/')[-1]}` (ncu --set full)\n")
            print("| kernel | " + " | ".join(n for _, n in METRICS) + " |")
            print("|---|" + "---|" * len(METRICS))
            for r in rows[2:]:
                vals = []
                for m, _ in METRICS:
                    i = hdr.index(m) if m in hdr else -1
                    vals.append(f"{r[i]} {units[i]}".strip() if i >= 0 else "n/a")
                print(f"| {r[hdr.index('Kernel Name')].split('(')[0][:40]} | " + " | ".join(vals) + " |")
            print()


if __name__ == "__main__":
    main()
