"""The C-ABI library on a CPU-only box: it loads, exports every function include/magus_replay.h declares,
validates configurations, derives the exact-equivalent thresholds on the host, and refuses to compute
without a GPU (there is no CPU fallback).  -m "not gpu"."""
import ctypes
import math
import os
import random
import subprocess

import numpy as np
import pytest

from paper_2502_03796_b200 import magus as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    names = M.header_functions()
    assert "magus_replay_create" in names and "magus_replay_run" in names and "magus_replay_results" in names
    out = subprocess.run(["nm", "-D", "--defined-only", M.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(M.LIB_PATH)
    for n in names:
        getattr(lib, n)
    assert M.abi_version() == 2


def test_library_is_sm100a_only():
    """Every kernel image in the library is sm_100a SASS (no PTX JIT, no other architecture)."""
    out = subprocess.run(["cuobjdump", "--list-elf", M.LIB_PATH], capture_output=True, text=True).stdout
    elves = [l for l in out.splitlines() if ".cubin" in l]
    assert elves and all("sm_100a" in l for l in elves), out
    ptx = subprocess.run(["cuobjdump", "--list-ptx", M.LIB_PATH], capture_output=True, text=True).stdout
    assert ".ptx" not in ptx


def test_sass_has_tma_and_no_fp64_division():
    """The replay kernel stages tiles with TMA (UTMALDG) and never divides per tick (no MUFU.RCP64H/DMUL
    Newton sequences): Alg. 1's division is replaced by exact-equivalent thresholds."""
    sass = subprocess.run(["cuobjdump", "-sass", M.LIB_PATH], capture_output=True, text=True).stdout
    funcs = sass.split("Function : ")
    replay = [f for f in funcs if f.startswith("_ZN5magus19magus_replay_kernel")]
    assert replay
    for f in replay:
        assert "UTMALDG" in f
        assert "MUFU.RCP64H" not in f and "DMUL" not in f


def test_generated_stage_macros_in_sync(tmp_path):
    """csrc/tick4_asm.cuh (the generated PTX stage blocks) is exactly what scripts/gen_tick4.py writes now."""
    out = tmp_path / "tick4_asm.cuh"
    subprocess.run(["python", os.path.join(ROOT, "scripts", "gen_tick4.py")], check=True, capture_output=True,
                   env={**os.environ, "MAGUS_GEN_OUT": str(out)})
    committed = open(os.path.join(ROOT, "paper_2502_03796_b200", "csrc", "tick4_asm.cuh")).read()
    assert out.read_text() == committed, "run python scripts/gen_tick4.py and rebuild"


def test_solo_batched_log_variants_in_library():
    """The default solo stage variants (BAL 24 / 25: the batched tune-flag log; 34 / 35 in open loop) and the fused
    kernel's batched-log build (LB) are compiled into the library for every register ring k <= 3."""
    sass = subprocess.run(["cuobjdump", "-res-usage", M.LIB_PATH], capture_output=True, text=True).stdout
    for k in (1, 2, 3):
        for bal in (24, 25, 34, 35):
            assert f"magus_replay_solo_kernelINS_11MagusTickerILi{k}ELb0EEELi8ELi3ELi{bal}EEE" in sass, (k, bal)
        assert f"magus_replay_fused_kernelINS_11MagusTickerILi{k}ELb0EEELi8ELi3ELb1ELi12ELb1ELb1EEE" in sass, k


def test_no_cuda_device_means_error_not_fallback():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("this box has a GPU")
    except ImportError:
        pass
    with pytest.raises(M.MagusError) as e:
        M.Replay(8, 100, [M.Policy()])
    assert e.value.status == M.ERR_CUDA


@pytest.mark.parametrize("bad,key", [(dict(deriv_ticks=0), "deriv_ticks"), (dict(dec_threshold=0.5), "dec_threshold"),
                                     (dict(inc_threshold=0.0), "inc_threshold"),
                                     (dict(tune_log_capacity=65), "tune_log_capacity"),
                                     (dict(high_freq_threshold=1.5), "high_freq_threshold"),
                                     (dict(kind=M.TDP_DEFAULT, tdp_margin=1.0), "tdp_margin"),
                                     (dict(kind=7), "kind")])
def test_config_validation_names_the_key(bad, key):
    """an invalid configuration is rejected before any device work, naming the key."""
    with pytest.raises(M.MagusError) as e:
        M.derive_thresholds(M.Policy(**bad), M.Model())
    assert e.value.status == M.ERR_CONFIG and key in str(e.value)
    with pytest.raises(M.MagusError) as e:
        M.derive_thresholds(M.Policy(), M.Model(f_min_ghz=3.0))
    assert "f_max_ghz" in str(e.value)


def _alg1_fires(d, L, th):
    return d / L > th


def test_dinc_ddec_are_exact_boundaries():
    """d*_inc is the largest double d with fl(d/L) <= theta_inc (Alg. 1 P:209 holds exactly iff d > d*);
    d*_dec the smallest with fl(d/L) >= theta_dec.  Checked with Python floats (IEEE doubles)
    at the boundary and one ulp either side, over random and paper-default parameters."""
    rng = random.Random(3)
    cases = [(1, 0.1, 1.0, -1.0), (3, 0.1, 1.0, -1.0), (8, 0.1, 0.5, -4.0)]
    cases += [(rng.randint(1, 64), rng.choice([0.1, 0.05, 0.3, 1.0]), rng.uniform(1e-3, 50), -rng.uniform(1e-3, 50))
              for _ in range(200)]
    for k, dt, inc, dec in cases:
        t = M.derive_thresholds(M.Policy(deriv_ticks=k, inc_threshold=inc, dec_threshold=dec), M.Model(sample_period_s=dt))
        L = k * dt
        assert t["L"] == L
        di, dd = t["dinc"], t["ddec"]
        assert not (di / L > inc) and (math.nextafter(di, math.inf) / L > inc)
        assert not (dd / L < dec) and (math.nextafter(dd, -math.inf) / L < dec)


def test_smin_and_tdp_boundaries():
    """s_min = min{s : fl(s/C) >= theta_hf} (Alg. 2); the paper's 0.6 of 10 gives 6.
    a*[f] = the smallest fp32 A with fl(P[f] + fl(c*A)) >= fl((1-m)*TDP)."""
    assert M.derive_thresholds(M.Policy(), M.Model())["s_min"] == 6
    for C in range(1, 65):
        for th in (0.1, 0.25, 0.5, 0.6, 0.7, 0.75, 0.9, 1.0, 1 / 3):
            s = M.derive_thresholds(M.Policy(tune_log_capacity=C, high_freq_threshold=th), M.Model())["s_min"]
            want = next((x for x in range(C + 1) if x / C >= th), C + 1)
            assert s == want, (C, th)
    m = M.Model()
    for tdp in (217.0, 230.0, 270.0, 400.0, 150.0):
        t = M.derive_thresholds(M.Policy(kind=M.TDP_DEFAULT, tdp_w=tdp), m)
        bound = (1.0 - 0.05) * tdp
        for P, a in ((t["P_lo"], t["astar_lo"]), (t["P_hi"], t["astar_hi"])):
            f = lambda A: (P + 0.5 * float(np.float32(A))) >= bound
            if math.isinf(a):
                assert not f(np.float32(np.finfo(np.float32).max))
            else:
                assert f(a)
                if a > 0:
                    assert not f(np.nextafter(np.float32(a), np.float32(0)))


def test_default_model_constants():
    """B_lo = fl32(20 * (0.8/2.2)) = 7.2727275; P_lo = 116 W, P_hi = 200 W (the K5 calibration)."""
    t = M.derive_thresholds(M.Policy(), M.Model())
    assert t["B_lo"] == float(np.float32(20 * (0.8 / 2.2))) and t["B_hi"] == 20.0
    assert (t["P_lo"], t["P_hi"]) == (116.0, 200.0)


def test_active_savings_host_matches_oracle():
    """NEXT-4: magus_active_savings on synthetic per-policy totals equals the oracle's job-level
    active savings (one trace per policy, so the job sums are the totals); errors as SPEC.md:435 says."""
    from oracle import oracle as O
    rng = np.random.default_rng(7)
    for _ in range(50):
        tot = np.zeros((3, M.N_TOTALS))
        tot[:, 0] = rng.uniform(100.0, 5000.0, 3)          # E
        tot[:, 2] = rng.uniform(1.0, 20.0, 3)              # T
        P = tot[:, 0] / tot[:, 2]
        p_idle = float(rng.uniform(0.0, 0.9) * min(P))
        for pol, base in ((0, 1), (2, 1), (1, 1)):
            got = M.active_savings(tot, pol, base, p_idle)
            want = O.active_savings_job([tot[pol, 0]], [tot[pol, 2]], [tot[base, 0]], [tot[base, 2]], p_idle)
            assert got == pytest.approx(want, rel=1e-12, abs=1e-15)
    tot = np.zeros((2, M.N_TOTALS))
    tot[:, 0], tot[:, 2] = (150.0, 200.0), (1.0, 1.0)
    assert M.active_savings(tot, 0, 1, 100.0)[0] == 0.5          # the paper's example
    for bad in ((0, 1, 250.0), (0, 2, 10.0), (0, 1, -1.0), (0, 1, 160.0)):
        with pytest.raises(M.MagusError):
            M.active_savings(tot, *bad)


def test_wallclock_flag_rejects_word_dump():
    """NEXT-1 (A32): the per-32-tick word dump has no meaning per round; the combination is refused at create,
    before any device work (so this holds on a CPU-only host too)."""
    with pytest.raises(M.MagusError) as e:
        M.Replay(8, 100, [M.Policy()], flags=M.F_WALLCLOCK | M.F_DUMP_WORDS)
    assert e.value.status == M.ERR_INVALID_ARG and "WALLCLOCK" in str(e.value)


@pytest.mark.parametrize("shape,knee", [(0, 1.0), (1, 0.5), (1, 0.25), (1, 1.0), (1, 0.9)])
def test_library_bandwidth_endpoints_equal_oracle(shape, knee):
    """The library's closed-loop bandwidths B_lo = fl32(bandwidth_at(f_min)), B_hi and powers P_lo, P_hi
    (magus_derive_thresholds, host side) equal the pinned oracle's SPEC.md:330-347 model for the Linear
    and the Saturating shapes (K14); the two sides share no code."""
    from oracle import oracle as O
    for e in (1.0, 2.5):
        th = M.derive_thresholds(M.Policy(), M.Model(bw_shape=shape, bw_knee=knee, p_exponent=e))
        om = O.Model(bw_shape=shape, bw_knee=knee, p_exponent=e)
        assert th["B_lo"] == np.float32(O.bandwidth_at(0.8, om))
        assert th["B_hi"] == np.float32(O.bandwidth_at(2.2, om))
        assert th["P_lo"] == O.pkg_power_at(0.8, om) and th["P_hi"] == O.pkg_power_at(2.2, om)
