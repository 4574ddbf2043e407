"""Summarise an ncu --set full report (one kernel) into the plain-text form
(ncu_summary.py plus the stall and instruction-mix tables)
kept under profiles/: headline metrics, then the warp-stall breakdown and
instruction mix from the source page.  Usage: ncu_stalls.py REPORT.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv",
                      "--print-units", "base"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
col = {k: i for i, k in enumerate(hdr)}
print("kernel:", vals[col["Kernel Name"]])
for m in METRICS:
    if m in col:
        print(f"  {m:64s} {vals[col[m]]:>22s} {units[col[m]]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(src)))
h, body = r[1], r[2:]
idx = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot, ops = collections.Counter(), collections.Counter()
for row in body:
    for k in stalls:
        try:
            tot[k] += int(row[idx[k]])
        except ValueError:
            pass
    t = row[idx["Source"]].strip().split()
    if t:
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += int(row[idx["Instructions Executed"]] or 0)
S = sum(tot.values()) or 1
print("warp stall sampling (all samples):")
for k, v in tot.most_common(10):
    print(f"  {k:28s} {100 * v / S:5.1f} %")
n = sum(ops.values()) or 1
print(f"instructions executed (warp-level): {n}")
for k, v in ops.most_common(14):
    print(f"  {k:10s} {100 * v / n:5.1f} %")
