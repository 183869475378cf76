#!/usr/bin/env python
"""SASS mix of the fused MAGUS + TDP kernel's steady stage loop (no GPU): per trace-sample instruction counts of the
backward-branch loop with 8 LDS.128 and the most DFMAs.  usage: python scripts/fused_sass.py <cubin-or-.so>"""
import re
import subprocess
import sys
from collections import Counter

sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", sass):
    if not f.startswith("_ZN5magus25magus_replay_fused"):
        continue
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
            nlds = sum("LDS.128" in x[1] for x in body)
            if nlds == 8 and (best is None or len(body) < len(best[2])):
                best = (lo, a, body)
    lo, a, body = best
    ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", o).split()[0] for _, o in body)
    spill = sum("LDL" in o or "STL" in o for _, o in body)
    print(f"{f.split()[0][:60]}: loop {hex(lo)}-{hex(a)}: {len(body)} instr -> {len(body) / 32:.2f} / sample; spills {spill}")
    print("   ", ", ".join(f"{k} {v / 32:.2f}" for k, v in ops.most_common(28)))
