#!/usr/bin/env python
"""Per-tick SASS instruction mix of the replay kernel's unrolled fast path (no GPU needed).

usage: python scripts/sass_stats.py [kernel-substring] [ticks-in-fast-path]
"""
import re
import subprocess
import sys
from collections import Counter

LIB = "paper_2502_03796_b200/lib/libmagus_replay.so"
PIPE = {  # coarse pipe classes (B300_MICROARCH.md: fma vs alu split; fp64; xu)
    "alu": ["FSEL", "FMNMX", "FSETP", "ISETP", "LOP3", "SEL", "PLOP3", "SHF", "VIMNMX", "IADD3", "VIADD", "PRMT",
            "P2R", "R2P", "IABS", "IMNMX", "LEA", "FLO", "BMSK", "SGXT"],
    "fma": ["IMAD", "FFMA", "FADD", "FMUL", "IADD"],
    "fp64": ["DADD", "DSETP", "DFMA", "DMUL", "DMNMX"],
    "xu": ["F2F", "POPC", "MUFU", "F2I", "I2F", "FRND"],
    "mem": ["LDS", "LDG", "STG", "STS", "LDL", "STL"],
}


def pipe_of(op):
    base = op.split(".")[0]
    for k, v in PIPE.items():
        if base in v:
            return k
    return "other"


def main():
    pat = sys.argv[1] if len(sys.argv) > 1 else "MagusTickerILi1ELb0"
    ticks = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    body = [f for f in funcs if pat in f.split("\n")[0] and "replay_kernel" in f.split("\n")[0]][0]
    lines = [l for l in body.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
    ops = [re.sub(r"^\s+/\*[0-9a-f]+\*/\s+", "", l).split(";")[0].strip() for l in lines]
    ops = [re.sub(r"^@!?U?P\w+\s+", "", o) for o in ops]
    # basic blocks: split at branch instructions and at jump targets (".L_x_NN:" labels)
    blocks, cur = [], []
    for l in body.split("\n"):
        if re.match(r"\s*\.L_x_\d+:", l):
            if cur:
                blocks.append(cur)
            cur = []
            continue
        if not re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
            continue
        o = re.sub(r"^\s+/\*[0-9a-f]+\*/\s+", "", l).split(";")[0].strip()
        o = re.sub(r"^@!?U?P\w+\s+", "", o)
        cur.append(o)
        if o.startswith(("BRA", "EXIT", "RET", "BRX", "CALL")):
            blocks.append(cur)
            cur = []
    if cur:
        blocks.append(cur)
    # the fast path: the block with the most LDS.128 tile reads (one per tick per lane = 4 chains)
    seg = max(blocks, key=lambda b: sum(1 for o in b if o.startswith("LDS.128")))
    ticks = 4 * sum(1 for o in seg if o.startswith("LDS.128"))
    c = Counter(o.split()[0] for o in seg)
    pc = Counter()
    for k, v in c.items():
        pc[pipe_of(k)] += v
    n = sum(c.values())
    print(f"{pat}: {len(ops)} SASS instr total; fast-path window {n} instr over {ticks} chain-ticks = "
          f"{n / ticks:.2f} / chain-tick")
    print("  by pipe: " + ", ".join(f"{k} {v / ticks:.2f}" for k, v in pc.most_common()))
    print("  top ops: " + ", ".join(f"{k} {v / ticks:.2f}" for k, v in c.most_common(18)))


if __name__ == "__main__":
    main()
