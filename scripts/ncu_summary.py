#!/usr/bin/env python
"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU).

    python scripts/ncu_summary.py full  gpurun_out/r3_nbody22.ncu-rep ... > profiles/x.md
    python scripts/ncu_summary.py launches gpurun_out/launches.csv > profiles/y.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def full(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(f"## {p}: no data\n")
            continue
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
            print(f"## {p}\n\nkernel: `{name[:120]}`\n")
            print("| metric | value | unit |\n|---|---|---|")
            for m in METRICS:
                if m in h:
                    i = h.index(m)
                    print(f"| {m} | {r[i]} | {units[i]} |")
            print()


def launches(paths):
    for p in paths:
        rows = list(csv.reader(open(p)))
        hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
        h = rows[hi]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        d = defaultdict(list)
        for r in rows[hi + 1:]:
            if len(r) > vi:
                d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in d.values())
        print(f"## {p} (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)\n")
        print("| kernel | launches | mean us | total us | share of listed time |\n|---|---|---|---|---|")
        for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
            print(f"| `{k[-70:]}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / 1e3:.1f} | "
                  f"{sum(v) / tot:.3f} |")
        print()


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2:])
