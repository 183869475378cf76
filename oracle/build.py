"""Build the CPU oracle shared library (TEST INFRASTRUCTURE ONLY).

g++ -O2 -ffp-contract=off: no FMA contraction, no fast-math, so every fp64
operation is the IEEE round-to-nearest result of the written expression
(reading A22).  `__graft_entry__.build()` calls this too: building
the checker is not using it.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["magus_oracle.cpp", "gen_oracle.cpp", "sample_oracle.cpp"]
LIB = os.path.join(HERE, "libmagus_oracle.so")


def build(force: bool = False) -> str:
    srcs = [os.path.join(HERE, s) for s in SOURCES] + [os.path.join(HERE, "oracle.h")]
    if not force and os.path.exists(LIB):
        newest = max(os.path.getmtime(s) for s in srcs)
        if os.path.getmtime(LIB) >= newest:
            return LIB
    cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-pthread", "-Wall", "-Wno-unused-function", "-o", LIB + ".tmp"]
    cmd += [os.path.join(HERE, s) for s in SOURCES]
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
