"""Build libmagus_replay.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo).

    python -m paper_2502_03796_b200._build [--force]
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libmagus_replay.so")
# the debug-check build (device-side bounds checks that trap, MAGUS_DEBUG_CHECKS=1; device_common.cuh), loaded only by
# tests/test_debug_checks.py through MAGUS_LIB_PATH
LIB_DEBUG = os.path.join(LIBDIR, "libmagus_replay_debug.so")
SOURCES = ["magus_replay.cu", "gen_traces.cu", "ingest.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _nccl_include() -> str:
    purelib = sysconfig.get_paths()["purelib"]
    cand = os.path.join(purelib, "nvidia", "nccl", "include")
    if os.path.exists(os.path.join(cand, "nccl.h")):
        return cand
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include"
    raise RuntimeError("nccl.h not found (torch's nvidia/nccl wheel or /usr/include)")


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "magus_replay.h"),
                                                               __file__]


def build(force: bool = False, verbose: bool = False, out: str | None = None, debug: bool = False) -> str:
    """Compile the library; `out` (or MAGUS_LIB_OUT) = another output path, for build-variant experiments;
    debug = the debug-check build (LIB_DEBUG)."""
    out = out or os.environ.get("MAGUS_LIB_OUT")
    if out:
        return _compile(out, verbose)
    lib = LIB_DEBUG if debug else LIB
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= max(os.path.getmtime(d) for d in _deps()):
        return lib
    return _compile(lib, verbose, ["-DMAGUS_DEBUG_CHECKS=1"] if debug else [])


def build_all(force: bool = False) -> None:
    """The release and the debug-check library, compiled concurrently."""
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(2) as ex:
        for f in [ex.submit(build, force, False, None, False), ex.submit(build, force, False, None, True)]:
            f.result()


def _compile(LIB: str, verbose: bool, extra: list | None = None) -> str:
    LIBDIR = os.path.dirname(os.path.abspath(LIB))
    os.makedirs(LIBDIR, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
                    "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", _nccl_include()]
    for key in ("MAGUS_TC", "MAGUS_NSTAGE"):
        if os.environ.get(key):
            flags += [f"-D{key}={int(os.environ[key])}"]
    flags += os.environ.get("MAGUS_DEFS", "").split()   # build-variant experiments, e.g. "-DMAGUS_SOLO_UNROLL=2"
    flags += extra or []
    if os.environ.get("MAGUS_PTXAS_VERBOSE"):
        flags += ["-Xptxas", "-v"]
    for src in SOURCES:
        obj = os.path.join(LIBDIR, os.path.splitext(os.path.basename(LIB))[0] + "_" + os.path.splitext(src)[0] + ".o")
        cmd = [nvcc, "-c", os.path.join(CSRC, src), "-o", obj] + flags
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = LIB + ".tmp"
    subprocess.check_call([nvcc, "-shared"] + ARCH + ["-o", tmp] + objs + ["-ldl"])
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    if "--debug" in sys.argv:
        print(build(force="--force" in sys.argv, verbose=True, debug=True))
    elif "--all" in sys.argv:
        build_all(force="--force" in sys.argv)
    else:
        print(build(force="--force" in sys.argv, verbose=True))
