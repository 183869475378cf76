"""The debug-check build (lib/libmagus_replay_debug.so: MAGUS_DEBUG_CHECKS=1, device_common.cuh): every chain-state,
ring and chain-total index and every shared-memory tile / scratch access of the replay kernels is checked against its
allocation, and a violation traps the kernel.  It stands in for compute-sanitizer's memcheck where that tool is not
available (profiles/r02_sanitize_closed.txt).  The CPU tests check that the build exists, exports the same C ABI and
reports its checks as compiled in; the GPU tests show that a failed check traps, and run scripts/sanitize_run.py (small
replays of every kernel family, each compared with the oracle) through the debug build."""
import ctypes
import os
import subprocess
import sys

import pytest

from paper_2502_03796_b200 import _build
from paper_2502_03796_b200 import magus as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = _build.LIB_DEBUG

needs_debug_lib = pytest.mark.skipif(not os.path.exists(DEBUG_LIB), reason="debug-check build not built "
                                     "(python -m paper_2502_03796_b200._build --debug)")


def _run(code, timeout=900):
    env = dict(os.environ, MAGUS_LIB_PATH=DEBUG_LIB)
    return subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=timeout)


@needs_debug_lib
def test_debug_build_exports_the_abi_and_has_checks():
    out = subprocess.run(["nm", "-D", "--defined-only", DEBUG_LIB], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    missing = [n for n in M.header_functions() if n not in exported]
    assert not missing, missing
    assert ctypes.CDLL(M.LIB_PATH).magus_debug_check_probe(0) == -1   # release build: checks compiled out


@pytest.mark.gpu
@needs_debug_lib
def test_debug_check_traps():
    """A failed MAGUS_CHECK traps the kernel (the probe launches one thread checking violate == 0); a passing check
    does not."""
    code = "from paper_2502_03796_b200 import magus as M; print(M.lib.magus_debug_check_probe({}))"
    ok = _run(code.format(0), 300)
    assert ok.returncode == 0 and ok.stdout.strip() == "0", ok.stdout + ok.stderr
    bad = _run(code.format(1), 300)
    assert bad.returncode == 0 and bad.stdout.strip() == "1", bad.stdout + bad.stderr


@pytest.mark.gpu
@needs_debug_lib
def test_every_kernel_family_under_debug_checks():
    """scripts/sanitize_run.py through the debug build: the solo (L stage and variant 2), fused MAGUS + TDP (12- and
    16-CTA builds), combined, multi-warp and wide (P / L / D stages) replay kernels, the pre-pass, the fix-up walks,
    totals, chunk sums with the one-rank NCCL exchange, the wall-clock kernels and the counter ingest -- each run
    compared with the oracle, no check trapped."""
    r = subprocess.run([sys.executable, "scripts/sanitize_run.py"], cwd=ROOT, capture_output=True, text=True,
                       timeout=1500, env=dict(os.environ, MAGUS_LIB_PATH=DEBUG_LIB))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ingest: ok" in r.stdout
    n = r.stdout.count(": ok")
    print(f"{n} cases ok under the debug-check build")
