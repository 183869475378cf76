#!/usr/bin/env python
"""SASS statistics of the unified-stage solo kernel (no GPU): the stage loop's instruction mix per chain-tick.
usage: python scripts/usolo_sass.py <cubin-or-.so> [K] [SYM 0|1]"""
import re
import subprocess
import sys
from collections import Counter

obj = sys.argv[1]
K = sys.argv[2] if len(sys.argv) > 2 else "1"
SYM = "Lb1" if (len(sys.argv) > 3 and sys.argv[3] == "1") or len(sys.argv) <= 3 else "Lb0"
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
f = [x for x in funcs if x.startswith(f"_ZN5magus25magus_replay_usolo_kernelINS_11MagusTickerILi{K}ELb0EEELi8ELi3EL{SYM[1:]}")][0]
ins = []
for l in f.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
print("total instructions", len(ins), " LDS.128:", sum("LDS.128" in o for _, o in ins))
for a, o in ins:
    t = re.search(r"BRA.*0x([0-9a-f]+)", o)
    if t and int(t.group(1), 16) < a:
        lo = int(t.group(1), 16)
        body = [x for x in ins if lo <= x[0] <= a]
        nlds = sum("LDS.128" in x[1] for x in body)
        if nlds >= 8:
            ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", o).split()[0] for _, o in body)
            print(f"loop {hex(lo)}-{hex(a)}: {len(body)} instr, {nlds} LDS.128 -> {len(body) / (4 * nlds):.2f} "
                  f"per chain-tick (whole loop incl. pipeline, fold, ragged path)")
            print("   ", ", ".join(f"{k} {v / (4 * nlds):.2f}" for k, v in ops.most_common(30)))
