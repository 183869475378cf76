#!/usr/bin/env python
"""Decode Volta+ control bits (stall, yield, barriers) of the replay kernel's fast-path block."""
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else "MagusTickerILi1ELb0"
show = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sass = subprocess.run(["cuobjdump", "-sass", "paper_2502_03796_b200/lib/libmagus_replay.so"], capture_output=True,
                      text=True).stdout
f = [x for x in re.split(r"\n\s+Function : ", sass) if pat in x.split("\n")[0] and "replay_kernel" in x.split("\n")[0]][0]
ins, cur = [], None
for line in f.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", line)
    if m:
        cur = [m.group(2), int(m.group(3), 16)]
        continue
    m2 = re.match(r"\s+/\* (0x[0-9a-f]+) \*/", line)
    if m2 and cur is not None:
        hi = int(m2.group(1), 16)
        cur.append(hi)
        ins.append(cur)
        cur = None
blocks, b = [], []
for op, lo, hi in ins:
    b.append((op, hi))
    if re.match(r"(@!?U?P\w+\s+)?(BRA|EXIT|BAR|SYNCS)", op):
        blocks.append(b)
        b = []
blocks.append(b)
fast = max(blocks, key=lambda bb: sum(1 for o, _ in bb if "LDS.128" in o))
n_lds = sum(1 for o, _ in fast if "LDS.128" in o)
stall = [((hi >> 41) & 0xF) for _, hi in fast]
waitm = [((hi >> 52) & 0x3F) for _, hi in fast]
print(f"fast block: {len(fast)} instr, {n_lds} LDS.128 ({4 * n_lds} chain-ticks); sum of stall cycles "
      f"{sum(stall)} -> {sum(stall) / (4 * n_lds):.1f} cycles per chain-tick for one warp alone; "
      f"{sum(1 for w in waitm if w)} instr wait on scoreboards")
if show:
    for (op, hi), s_, w in zip(fast[:show], stall, waitm):
        print(f"  s{s_:2d} w{w:02x}  {op}")
