#!/usr/bin/env python
"""Summarise an exported ncu raw page (`ncu -i X.ncu-rep --page raw --csv > X_raw.csv`, written on the GPU box so the
report itself need not travel back) into a profiles/ text file: time, DRAM bytes vs the algorithmic bytes, issue,
pipes, occupancy, warp stalls, lane instructions per unit.
usage: python scripts/profile_from_csv.py RAW.csv OUT.txt "title" ALGO_BYTES UNITS [bench.json]"""
import csv
import json
import sys

raw, out, title, alg, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]), float(sys.argv[5])
rows = list(csv.reader(open(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed_op_tma_ld.sum"]
lines = [f"# {title}", ""]
for k in keys:
    if k in d:
        lines.append(f"{k:75s} {d[k][0]:>24s} {d[k][1]}")
st = sorted(((k, float(d[k][0].replace(",", ""))) for k in d
             if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
             and d[k][0].replace(",", "").replace(".", "").isdigit()), key=lambda t: -t[1])
lines += ["", "warp stalls per issued instruction:"]
lines += [f"   {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:40s} {x:7.3f}"
          for k, x in st[:10] if x > 0.02]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rb = float(d["dram__bytes_read.sum"][0].replace(",", "")) * UNIT[d["dram__bytes_read.sum"][1]]
wb = float(d["dram__bytes_write.sum"][0].replace(",", "")) * UNIT[d["dram__bytes_write.sum"][1]]
inst = float(d["smsp__inst_executed.sum"][0].replace(",", ""))
lines += ["", f"DRAM traffic per launch {rb + wb:.4e} B vs algorithmic {alg:.4e} B: x{(rb + wb) / alg:.3f}",
          f"lane instructions per unit: {inst * 32 / units:.2f} ({inst:.4e} warp instructions x 32 / {units:.4e} units)"]
if len(sys.argv) > 6:
    b = json.load(open(sys.argv[6]))
    lines.append(f"bench roofline (live CUDA events): {json.dumps(b['roofline'])}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[-3:]))
