#!/usr/bin/env python
"""SASS statistics of the wide replay kernel's steady 32-tick block (no GPU): the backward branch whose body holds
the most DADDs is the stage loop; per chain-tick instruction mix = body / 32.
usage: python scripts/wide_sass.py <cubin-or-.so> [K] [LV]"""
import re
import subprocess
import sys
from collections import Counter

obj = sys.argv[1]
K = sys.argv[2] if len(sys.argv) > 2 else "1"
LV = sys.argv[3] if len(sys.argv) > 3 else "0"
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
f = [x for x in funcs if x.startswith(f"_ZN5magus24magus_replay_wide_kernelILi{K}ELi1ELi{LV}E")][0]
ins = []
for l in f.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for a, o in ins:
    t = re.search(r"BRA.*0x([0-9a-f]+)", o)
    if t and int(t.group(1), 16) < a:
        lo = int(t.group(1), 16)
        body = [x for x in ins if lo <= x[0] <= a]
        nd = sum(" DADD" in " " + x[1] or x[1].startswith("DADD") for x in body)
        if best is None or nd > best[0]:
            best = (nd, lo, a, body)
nd, lo, a, body = best
# the steady branch: the span between the first and last DADD of the stage loop region with 96 DADDs (3 per tick)
ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", o).split()[0] for _, o in body)
print(f"loop {hex(lo)}-{hex(a)}: {len(body)} instr, {nd} DADD")
print("   ", ", ".join(f"{k} {v}" for k, v in ops.most_common(30)))
