#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into the small
text files kept under profiles/.

    python scripts/ncu_summary.py report.ncu-rep  > profiles/rNN_x.txt
    python scripts/ncu_summary.py launches.csv     > profiles/rNN_launches.txt
"""

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f"kernel: {r[head.index('Kernel Name')]}")
        for k in KEYS:
            if k in head:
                i = head.index(k)
                print(f"  {k:62s} {r[i]:>14s} {units[i]}")
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    for r in csv.reader(io.StringIO(det)):
        if len(r) > 15 and r[13] in ("Warp Cycles Per Issued Instruction",
                                      "Achieved Occupancy", "Duration",
                                      "DRAM Throughput", "Memory Throughput"):
            print(f"  [{r[12]}] {r[13]}: {r[15]} {r[14]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    print(f"{'launches':>8s} {'mean ns':>10s} {'share':>7s}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v):10.0f} {sum(v) / total:7.1%}  "
              f"{k[:110]}")


if __name__ == "__main__":
    p = sys.argv[1]
    (rep if p.endswith(".ncu-rep") else launches)(p)
