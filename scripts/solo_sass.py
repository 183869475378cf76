#!/usr/bin/env python
"""SASS statistics of the solo replay kernel's stage blocks (no GPU): per-chain-tick instruction mix of the
steady-state block and the local-memory (spill) instructions inside the stage loops.
usage: python scripts/solo_sass.py <object-or-.so> [K] [BAL 0|1]"""
import re
import subprocess
import sys
from collections import Counter

obj = sys.argv[1]
K = sys.argv[2] if len(sys.argv) > 2 else "1"
BAL = sys.argv[3] if len(sys.argv) > 3 else "1"   # 1: the pipe-balanced stage variant
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
f = [x for x in funcs if x.startswith(f"_ZN5magus24magus_replay_solo_kernelINS_11MagusTickerILi{K}ELb0EEELi8ELi3ELi{BAL}")][0]
ins = []
for l in f.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
loops = []
for a, o in ins:
    t = re.search(r"BRA.*0x([0-9a-f]+)", o)
    if t and int(t.group(1), 16) < a:
        lo = int(t.group(1), 16)
        body = [x for x in ins if lo <= x[0] <= a]
        nlds = sum("LDS.128" in x[1] for x in body)
        if nlds >= 8:
            loops.append((lo, a, body, nlds))
for lo, a, body, nlds in loops:
    ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", o).split()[0] for _, o in body)
    spill = [(hex(x), o) for x, o in body if "LDL" in o or "STL" in o]
    print(f"loop {hex(lo)}-{hex(a)}: {len(body)} instr, {nlds} LDS.128 -> {len(body) / (4 * nlds):.2f} / chain-tick;"
          f" spills in loop: {len(spill)}")
    print("   ", ", ".join(f"{k} {v / (4 * nlds):.2f}" for k, v in ops.most_common(24)))
