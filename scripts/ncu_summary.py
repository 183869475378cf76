#!/usr/bin/env python
"""Summarise an ncu report of the replay kernel: time, DRAM bytes, pipe use, issue, stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__cycles_active.avg"]
for k in keys:
    if k in d:
        print(f"{k:70s} {d[k][0]:>18s} {d[k][1]}")
stalls = [(k, float(d[k][0].replace(",", ""))) for k in d
          if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio")]
stalls = [(k, x) for k, x in stalls if x > 0.05]
print("warp stall reasons (cycles per issued instruction):")
for k, x in sorted(stalls, key=lambda t: -t[1])[:12]:
    print(f"   {k.replace('smsp__average_warp_latency_issue_stalled_', ''):50s} {x:8.2f}")
