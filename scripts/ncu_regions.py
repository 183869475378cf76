#!/usr/bin/env python
"""Executed-instruction regions of one kernel from an `ncu --set full --import-source on` report (no GPU
needed): consecutive SASS lines with the same execution count form a region; prints the largest regions
with their share of executed instructions and of warp-stall samples.

usage: python scripts/ncu_regions.py <report.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
data = rows[2:]
ia, isamp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ia]) for r in data)
samp = max(1, sum(int(r[isamp]) for r in data))
regions, cur = [], None
for i, r in enumerate(data):
    c, s = int(r[ia]), int(r[isamp])
    if cur and cur[2] == c:
        cur[1], cur[3], cur[4] = i, cur[3] + c, cur[4] + s
    else:
        if cur:
            regions.append(cur)
        cur = [i, i, c, c, s]
regions.append(cur)
print(f"{rows[0][1][:100]}: {tot} warp-instructions executed, {len(data)} SASS lines")
for a, b, c, t, s in sorted(regions, key=lambda x: -x[3])[:top]:
    print(f"  lines {a:5d}-{b:5d} ({b - a + 1:4d} instr) x {c:8d} = {100 * t / tot:5.1f}% instr, {100 * s / samp:5.1f}% "
          f"stall samples | {data[a][1].strip()[:48]}")
