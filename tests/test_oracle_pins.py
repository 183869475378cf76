"""Pins for the CPU oracle.  -m "not gpu".

Each test checks the oracle against something other than itself: a value the
paper prints, a hand derivation, a closed form, an invariant, or an
independent brute force.  A plausible mistake in the oracle (a dropped term, a
flipped comparison, an off-by-one FIFO, a wrong initial level) fails one of
them; the docstrings say which.
"""
import json
import math
import os
import random

import numpy as np
import pytest

from oracle import oracle as O
from tests import _bruteforce as BF

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CAUSE = {0: "HOLD", 1: "INC", 2: "DEC"}


def cause_of(code):
    if code & 8:
        return "LOCK"
    return CAUSE[(code >> 4) & 3]


# --------------------------------------------------------------------------- K1: Alg. 2 exhaustively

def test_alg2_exhaustive_c10():
    """K1: all 2^10 logs at the paper's 0.6: True iff popcount >= 6 -- the boundary is
    inclusive (P:230 '>='), so exactly six flags in ten lock.  A '>' bug fails at popcount 6."""
    for v in range(1 << 10):
        flags = [(v >> i) & 1 for i in range(10)]
        assert O.alg2(0.6, flags) == (sum(flags) >= 6), flags


def test_alg2_spec_examples_and_ratios():
    """SPEC.md:177-179 examples; ratio thresholds 0.75 of 4 and 0.7 of 10 (K1 s_min cases)."""
    assert O.alg2(0.6, [1, 1, 1, 1, 1, 1, 0, 0, 0, 0]) is True
    assert O.alg2(0.6, [0] * 10) is False
    assert O.alg2(0.6, [1] + [0] * 9) is False
    assert [O.alg2(0.75, [1] * s + [0] * (4 - s)) for s in range(5)] == [False, False, False, True, True]
    assert [O.alg2(0.6, [1] * s + [0] * (5 - s)) for s in range(6)] == [False] * 3 + [True] * 3
    assert [O.alg2(0.7, [1] * s + [0] * (10 - s)) for s in range(11)] == [False] * 7 + [True] * 4


def test_alg2_uses_len_not_capacity():
    """Alg. 2 divides by len(uncore_tune_ls): a partial log of one flag gives 1/1 = 1.0."""
    assert O.alg2(0.6, [1]) is True
    assert O.alg2(0.6, [1, 0]) is False


# --------------------------------------------------------------------------- K2: Alg. 1 boundaries

def test_alg1_strict_boundaries():
    """K2: derivative exactly equal to the threshold holds (strict > / <).
    fl(0.1/0.1) = 1.0 -> Hold; one ulp more -> Increase; mirrored for Decrease."""
    L = 0.1
    assert O.alg1(1.0, -1.0, [0.0, 0.1], L) == 0
    assert O.alg1(1.0, -1.0, [0.0, math.nextafter(0.1, 1.0)], L) == 1
    assert O.alg1(1.0, -1.0, [0.1, 0.0], L) == 0
    assert O.alg1(1.0, -1.0, [math.nextafter(0.1, 1.0), 0.0], L) == -1


def test_alg1_spec_examples():
    """constant -> Hold; 1e9 -> 2e10 over 1 s at 1e9 -> Increase; reverse -> Decrease;
    only the first and last entries of the list matter (P:207 ls[-1] - ls[0])."""
    assert O.alg1(1e9, -1e9, [5e9, 5e9, 5e9], 1.0) == 0
    assert O.alg1(1e9, -1e9, [1e9, 3e10, 0.0, 2e10], 1.0) == 1
    assert O.alg1(1e9, -1e9, [2e10, 0.0, 5e10, 1e9], 1.0) == -1
    assert O.alg1(1e9, -1e9, [0.0, 1e9], 1.0) == 0          # derivative == inc_threshold


def test_alg1_random_against_python_float():
    """Alg. 1 on random doubles equals the same two-line definition evaluated by Python floats."""
    rng = random.Random(7)
    for _ in range(2000):
        ls = [rng.uniform(0, 20) for _ in range(rng.randint(2, 9))]
        inc, dec, L = rng.uniform(0.01, 5), -rng.uniform(0.01, 5), rng.choice([0.1, 0.2, 0.3, 0.8])
        d = (ls[-1] - ls[0]) / L
        assert O.alg1(inc, dec, ls, L) == (1 if d > inc else (-1 if d < dec else 0))


# --------------------------------------------------------------------------- K4: hand-computed traces

def _worked_cases():
    return json.load(open(os.path.join(GOLD, "worked_traces.json")))


def _model_from_common(c):
    return O.Model(sample_period_s=c["sample_period_s"], bw_max_gbps=c["bw_max_gbps"], f_min_ghz=c["f_min_ghz"],
                   f_max_ghz=c["f_max_ghz"], p_pkg_idle_w=c["p_pkg_idle_w"], p_core_active_w=c["p_core_active_w"],
                   p_uncore_min_w=c["p_uncore_min_w"], p_uncore_max_w=c["p_uncore_max_w"],
                   p_gpu_active_w=c["p_gpu_active_w"])


@pytest.mark.parametrize("case", _worked_cases()["cases"], ids=lambda c: c["name"])
def test_worked_traces(case):
    """K4: per-tick level, tune flag and cause, and the totals, equal the hand derivation
    (tests/golden/worked_traces.json, Alg. 1/2 and S3.2)."""
    common = _worked_cases()["common"]
    model = _model_from_common(common)
    pol = O.Policy(deriv_ticks=case["k"], inc_threshold=common["inc_threshold"],
                   dec_threshold=common["dec_threshold"], tune_log_capacity=case["C"],
                   high_freq_threshold=case["high_freq_threshold"])
    res, codes = O.replay(np.array(case["D"], np.float32), common["w"], pol, model, codes=True)
    level = "".join("H" if c >> 7 else "L" for c in codes)
    events = "".join("-" if not (c >> 1) & 1 else str((c >> 2) & 1) for c in codes)
    assert level == case["level"]
    assert events == case["events"]
    assert [cause_of(c) for c in codes] == case["causes"]
    for key in ("transitions", "tune_events", "lock_ticks", "n_thr"):
        assert res[key] == case[key], key
    for key in ("T", "E", "E_pkg", "EDP", "slowdown", "energy_saving", "edp_saving", "pkg_power_saving"):
        if key in case:
            assert res[key] == pytest.approx(case[key], rel=1e-9, abs=1e-12), key


# --------------------------------------------------------------------------- K5: calibration closed form

def test_unet_calibration_closed_form():
    """K5: static f_min vs static f_max on a constant trace reproduces the paper's UNet case study
    (pkg power -42%, energy -13%, time +23%).  With w = 0.5 and B_lo = 8, demand
    D = 11.68 gives w + (1-w) D/B_lo = 1.23; P_lo/P_hi = 116/200 = 0.58; P_gpu = 87 = 0.435 P_hi,
    so energy ratio (0.58+0.435)*1.23/1.435 = 0.870.  A wrong dilation formula or a missing GPU
    energy term moves these by whole percentage points."""
    paper = json.load(open(os.path.join(GOLD, "paper_numbers.json")))["unet_min_vs_max"]
    model = O.Model(bw_max_gbps=22.0)
    D = np.full(100, 11.68, np.float32)
    smin, _ = O.replay(D, 0.5, O.Policy(kind=O.STATIC_MIN), model)
    smax, _ = O.replay(D, 0.5, O.Policy(kind=O.STATIC_MAX), model)
    assert smax["slowdown"] == pytest.approx(0.0, abs=1e-12)
    assert smin["slowdown"] == pytest.approx(paper["time_increase"], abs=1e-6)
    assert 1 - (smin["E_pkg"] / smin["T"]) / (smax["E_pkg"] / smax["T"]) == pytest.approx(paper["pkg_power_saving"], abs=1e-9)
    assert 1 - smin["E"] / smax["E"] == pytest.approx(paper["energy_saving"], abs=1e-6)
    assert smin["energy_saving"] == pytest.approx(paper["energy_saving"], abs=1e-6)


def test_static_max_closed_form():
    """K6: STATIC_MAX is never throttled (D <= bw_max), never transitions; T = N*Delta,
    E = (P_hi + P_gpu) * N * Delta (SPEC.md:363 lower bound)."""
    rng = np.random.default_rng(3)
    D = rng.uniform(0, 20, 500).astype(np.float32)
    r, codes = O.replay(D, 0.7, O.Policy(kind=O.STATIC_MAX), codes=True)
    assert r["transitions"] == 0 and r["n_thr"] == 0 and r["n_hi"] == 500
    assert r["T"] == pytest.approx(50.0, rel=1e-12)
    assert r["E"] == pytest.approx((200 + 87) * 50.0, rel=1e-12)
    assert np.all(codes == 0x81)


# --------------------------------------------------------------------------- K6: invariants

POLICIES = [
    O.Policy(),
    O.Policy(deriv_ticks=2, inc_threshold=0.5, dec_threshold=-0.5, high_freq_threshold=0.4),
    O.Policy(deriv_ticks=4, inc_threshold=4.0, dec_threshold=-4.0, high_freq_threshold=0.7),
    O.Policy(deriv_ticks=3, tune_log_capacity=4, high_freq_threshold=0.75),
    O.Policy(deriv_ticks=1, tune_log_capacity=64, high_freq_threshold=0.5),
    O.Policy(deriv_ticks=8, tune_log_capacity=1, high_freq_threshold=1.0),
    O.Policy(kind=O.TDP_DEFAULT, tdp_w=217.0),
    O.Policy(kind=O.STATIC_MIN),
    O.Policy(kind=O.STATIC_MAX),
]


def _random_trace(rng, n):
    kind = rng.integers(0, 4)
    if kind == 0:
        return rng.uniform(0, 20, n).astype(np.float32)
    if kind == 1:
        return np.where((np.arange(n) // rng.integers(1, 30)) % 2 == 0, rng.uniform(0.5, 4), rng.uniform(10, 19)).astype(np.float32)
    if kind == 2:
        return (np.round(rng.uniform(0, 20, n) * 4) / 4).astype(np.float32)
    return np.repeat(rng.uniform(0, 20, n // 7 + 1), 7)[:n].astype(np.float32)


def test_invariants_random():
    """K6: levels only f_min/f_max; Alg. 2 true => command is
    max; a tune flag is pushed on every ready tick, locked or not, starting at t = k; no policy beats
    static max in time; throttling only at f_min; transition count = number of level changes."""
    rng = np.random.default_rng(11)
    for trial in range(60):
        n = int(rng.integers(1, 400))
        D = _random_trace(rng, n)
        w = float(np.float32(rng.uniform(0.5, 0.95)))
        for pol in POLICIES:
            r, c = O.replay(D, w, pol, codes=True)
            cmd, ready, hf, thr, lvl = c & 1, (c >> 1) & 1, (c >> 3) & 1, (c >> 6) & 1, c >> 7
            assert np.all(cmd[hf == 1] == 1)
            if pol.kind == O.MAGUS:
                assert np.all(ready == (np.arange(n) >= pol.deriv_ticks))
                assert r["tune_events"] == int(((c >> 2) & 1).sum())
                assert r["lock_ticks"] == int(hf.sum())
                assert np.all(hf[: pol.deriv_ticks + pol.tune_log_capacity - 1] == 0)   # A8: full log required
            else:
                assert not ready.any() and not hf.any()
            assert np.all(thr[lvl == 1] == 0)
            assert r["n_thr"] == int(thr.sum()) and r["n_hi"] == int(lvl.sum())
            assert np.all(lvl[1:] == cmd[:-1])                                            # A15
            assert r["transitions"] == int((cmd != lvl).sum())
            assert r["T"] >= r["T_base"] * (1 - 1e-12)
            assert r["E"] == pytest.approx(r["E_pkg"] + 87.0 * r["T"], rel=1e-9)


def test_initial_levels():
    """A10: MAGUS and STATIC_MIN start at f_min, STATIC_MAX and the Intel default at f_max."""
    D = np.full(5, 3.0, np.float32)
    first = {p.kind: O.replay(D, 0.5, p, codes=True)[1][0] >> 7 for p in
             [O.Policy(), O.Policy(kind=O.STATIC_MIN), O.Policy(kind=O.STATIC_MAX), O.Policy(kind=O.TDP_DEFAULT)]}
    assert first == {O.MAGUS: 0, O.STATIC_MIN: 0, O.STATIC_MAX: 1, O.TDP_DEFAULT: 1}


# --------------------------------------------------------------------------- K7 / K8 / K9: behaviour

def test_convergence_on_constant_input():
    """K7: constant throughput -> after warm-up no flags, no transitions, level fixed at f0 (MAGUS
    f_min), both below and above B_lo (above: the closed-loop blind spot, ex5 / A14)."""
    for level in (1.0, 3.5, 7.0, 12.0, 19.9):
        r, c = O.replay(np.full(300, level, np.float32), 0.6, O.Policy(), codes=True)
        assert r["transitions"] == 0 and r["tune_events"] == 0 and r["n_hi"] == 0


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_bounded_reaction_clean_step(k):
    """K8: a clean step below B_lo (2 -> 6 GB/s at t0, |dA|/(k*Delta) >> 1) fires Increase at t0 and
    the level is max from t0+1: one tick of reaction.  The step is seen for exactly k ticks, so
    k flags; with C = 10, s_min = 6 > k no lock; one transition up, then one down on the falling edge."""
    t0 = 40
    D = np.array([2.0] * t0 + [6.0] * 60 + [2.0] * 60, np.float32)
    r, c = O.replay(D, 0.5, O.Policy(deriv_ticks=k), codes=True)
    sig = (c >> 4) & 3
    assert list(np.nonzero(sig == 1)[0]) == list(range(t0, t0 + k))
    assert (c[t0] >> 7) == 0 and all((c[t] >> 7) == 1 for t in range(t0 + 1, t0 + 61))
    assert list(np.nonzero(sig == 2)[0]) == list(range(t0 + 60, t0 + 60 + k))
    assert r["transitions"] == 2 and r["tune_events"] == 2 * k and r["lock_ticks"] == 0


def test_throttled_rising_edge_sees_k_plus_one_flags():
    """K8 (ex6 generalised): a rising edge above B_lo seen at f_min produces k+1 Increase flags,
    because the un-throttling jump B_lo -> D is observed once more after the switch."""
    for k in (1, 2, 3):
        D = np.array([2.0] * 20 + [12.0] * 40, np.float32)
        r, c = O.replay(D, 0.5, O.Policy(deriv_ticks=k, tune_log_capacity=10), codes=True)
        assert r["tune_events"] == k + 1 and r["transitions"] == 1


def test_toggle_suppression():
    """K9 (SPEC AC4): toggling every tick across B_lo, k = 1, C = 10, 0.6: flags every
    tick from t = 1, lock from t = k + C - 1 = 10, at most C - 1 = 9 transitions before the lock,
    none while it persists; after toggling stops the lock releases after C - s_min + 1 = 5 quiet
    ticks and the level stays at max (post-lock stickiness)."""
    n_tog = 200
    D = np.array([2.0, 12.0] * (n_tog // 2) + [12.0] * 50, np.float32)
    r, c = O.replay(D, 0.5, O.Policy(), codes=True)
    hf = (c >> 3) & 1
    assert hf[:10].sum() == 0 and np.all(hf[10:n_tog] == 1)
    assert r["transitions"] <= 9
    cmd = c & 1
    assert np.all(cmd[10:] == 1)
    # release: the first quiet tick is t = n_tog (12 -> 12), the log drops below 6 ones after 5 quiet ticks
    assert np.all(hf[n_tog:n_tog + 4] == 1) and np.all(hf[n_tog + 4:] == 0)


def test_even_k_aliasing_on_period_two():
    """K9 corner: with even k a period-2 oscillation has A_t - A_{t-k} = 0 -> no flags, no transitions."""
    D = np.array([2.0, 6.0] * 100, np.float32)
    for k in (2, 4, 8):
        r, _ = O.replay(D, 0.5, O.Policy(deriv_ticks=k))
        assert r["tune_events"] == 0 and r["transitions"] == 0


def test_transitions_before_first_lock_bounded():
    """K9: for any input at most C - 1 transitions happen before the log first fills (ticks k..k+C-2)."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        D = rng.uniform(0, 20, 64).astype(np.float32)
        for C in (2, 4, 10):
            _, c = O.replay(D, 0.5, O.Policy(tune_log_capacity=C), codes=True)
            first = 1 + C - 1
            trans = ((c & 1) != (c >> 7))[:first]
            assert trans.sum() <= C - 1


# --------------------------------------------------------------------------- K10 / K12: brute force

def test_full_prefix_bruteforce_and_fsum():
    """K10 + K12: the oracle's FIFO loop emits exactly the codes of an independent re-evaluation of
    Alg. 1/2 over the full observed prefix at every tick (AC3), and its running fp64
    sums of energy/time agree with exactly-rounded math.fsum of the same per-tick terms to 1e-12."""
    rng = np.random.default_rng(1234)
    specs = [(1, 1.0, -1.0, 10, 0.6), (2, 0.5, -0.5, 10, 0.4), (4, 2.0, -2.0, 10, 0.7), (3, 1.0, -1.0, 4, 0.75),
             (5, 0.25, -3.0, 7, 0.5), (8, 4.0, -4.0, 10, 0.5), (1, 1.0, -1.0, 1, 1.0), (2, 1.0, -1.0, 33, 0.6)]
    for trial in range(40):
        n = int(rng.integers(1, 1000))
        D = _random_trace(rng, n)
        w = float(np.float32(rng.uniform(0.5, 0.95)))
        for (k, inc, dec, C, hf) in specs:
            rows, sums = BF.replay_prefix(D, w, k, inc, dec, C, hf)
            r, codes = O.replay(D, w, O.Policy(deriv_ticks=k, inc_threshold=inc, dec_threshold=dec,
                                               tune_log_capacity=C, high_freq_threshold=hf), codes=True)
            assert np.array_equal(codes, BF.rows_to_codes(rows)), (trial, k, C)
            for key in ("T", "E_pkg", "E"):
                assert r[key] == pytest.approx(sums[key], rel=1e-12), key
        for kind, pol in (("tdp", O.Policy(kind=O.TDP_DEFAULT, tdp_w=217.0)), ("static_min", O.Policy(kind=O.STATIC_MIN))):
            rows, sums = BF.replay_prefix(D, w, 1, 1, -1, 10, 0.6, kind=kind, tdp=217.0)
            r, codes = O.replay(D, w, pol, codes=True)
            assert np.array_equal(codes, BF.rows_to_codes(rows)), kind
            assert r["E"] == pytest.approx(sums["E"], rel=1e-12)


# --------------------------------------------------------------------------- K11: scale equivariance

def test_power_of_two_scale_equivariance():
    """K11 (S:211 restricted to exact scalings): multiplying D, bw_max and both thresholds by 2^j leaves
    every code unchanged.  (S:211 states it for any constant, which holds only in exact arithmetic.)"""
    rng = np.random.default_rng(9)
    for trial in range(20):
        D = _random_trace(rng, 300)
        base, c0 = O.replay(D, 0.6, O.Policy(deriv_ticks=2), codes=True)
        for j in (-3, 1, 4):
            s = 2.0 ** j
            m = O.Model(bw_max_gbps=20.0 * s)
            _, cj = O.replay((D * np.float32(s)).astype(np.float32), 0.6,
                             O.Policy(deriv_ticks=2, inc_threshold=s, dec_threshold=-s), m, codes=True)
            assert np.array_equal(c0, cj)


# --------------------------------------------------------------------------- baselines and metrics

def test_tdp_default_spec_examples():
    """well below the bound -> f_max; pkg+DRAM 490 W >= 0.95*500 -> f_min; a GPU-dominant
    trace never nearing TDP stays at max for the whole run (P:282 'remain at its maximum')."""
    model = O.Model(p_pkg_idle_w=200.0, p_core_active_w=80.0, p_uncore_min_w=10.0, p_uncore_max_w=20.0,
                    dram_w_per_gbps=10.0)   # P_hi = 300 W; + 10 W per GB/s of DRAM traffic
    pol = O.Policy(kind=O.TDP_DEFAULT, tdp_w=500.0, tdp_margin=0.05)
    _, c = O.replay(np.array([0.0, 0.0], np.float32), 0.5, pol, model, codes=True)
    assert list(c & 1) == [1, 1]                  # 300 W < 475 W
    _, c = O.replay(np.array([19.0, 0.0, 0.0], np.float32), 0.5, pol, model, codes=True)
    assert list(c & 1) == [0, 1, 1]               # 300 + 190 = 490 >= 475 -> f_min, then reverts
    rng = np.random.default_rng(0)
    r, c = O.replay(rng.uniform(0, 20, 1000).astype(np.float32), 0.5, O.Policy(kind=O.TDP_DEFAULT, tdp_w=270.0),
                    codes=True)
    assert np.all(c & 1) and r["transitions"] == 0


def test_tdp_217_toggles_only_at_high_throughput():
    """cfg 5 reading: at 217 W the bound is 206.15 W; at f_max 200 + 0.5 A crosses it once A >= 12.3,
    never at f_min (116 + 0.5*A <= 126) -> memory-heavy stretches toggle max/min."""
    D = np.array([5.0] * 10 + [15.0] * 10, np.float32)
    _, c = O.replay(D, 0.5, O.Policy(kind=O.TDP_DEFAULT, tdp_w=217.0), codes=True)
    assert list(c[:10] & 1) == [1] * 10
    assert list(c[10:] & 1) == [0, 1] * 5


def test_metrics_spec_examples():
    """S:410-445 metric definitions, exercised through the oracle's results: slowdown = T/T_b - 1,
    savings = 1 - x/x_b, and the EDP composition identity edp_saving = 1 - (1-b)(1+a)."""
    case = [c for c in _worked_cases()["cases"] if c["name"] == "ex2"][0]
    common = _worked_cases()["common"]
    r, _ = O.replay(np.array(case["D"], np.float32), 0.5,
                    O.Policy(tune_log_capacity=4, high_freq_threshold=0.75), _model_from_common(common))
    a, b = r["slowdown"], r["energy_saving"]
    assert r["edp_saving"] == pytest.approx(1 - (1 - b) * (1 + a), rel=1e-12)
    assert r["T_base"] == pytest.approx(0.8) and r["E_base"] == pytest.approx(229.6)


def test_invalid_samples_rejected():
    """A17: negative, NaN, +inf or > bw_max samples are an error at the first offending tick."""
    for bad, pos in ((-1.0, 3), (float("nan"), 0), (float("inf"), 7), (20.5, 5)):
        D = np.full(10, 3.0, np.float32)
        D[pos] = bad
        r, _ = O.replay(D, 0.5, O.Policy())
        assert r["status"] == 2 and r["err_tick"] == pos
    r, _ = O.replay(np.array([0.0, -0.0, 20.0], np.float32), 0.5, O.Policy())
    assert r["status"] == 0


def test_digest_definition():
    """DESIGN.md s5 digest: order-independent sum over 32-tick blocks; a single flipped bit changes it;
    zero-padding of the partial last block equals explicitly padding with zero bits."""
    rng = np.random.default_rng(2)
    cmd = rng.integers(0, 2, 100).astype(np.uint8)
    ev = rng.integers(0, 2, 100).astype(np.uint8)
    d = O.digest(cmd, ev)
    # 100 ticks = 4 blocks, the last one partial; explicit zero bits up to 128 ticks give the same 4 words
    assert O.digest(np.r_[cmd, np.zeros(28, np.uint8)], np.r_[ev, np.zeros(28, np.uint8)]) == d
    for t in (0, 31, 32, 99):
        c2 = cmd.copy(); c2[t] ^= 1
        assert O.digest(c2, ev) != d
        e2 = ev.copy(); e2[t] ^= 1
        assert O.digest(cmd, e2) != d


# --------------------------------------------------------------------------- NEXT-4: active savings

def test_active_saving_paper_example():
    """P:401 worked example: total power 200 W -> 150 W with 100 W idle power is a 50% active saving."""
    g = json.load(open(os.path.join(GOLD, "paper_numbers.json")))["active_power_example"]
    assert O.active_saving(g["p"], g["p_base_w"], g["p_idle_w"]) == g["active_saving"]


def test_active_saving_properties():
    """p_idle = 0 reduces to the plain power saving; p = p_base gives 0; a common positive
    rescaling of the watts changes nothing (powers of two: exact); a baseline without active power or a power
    below idle is an error."""
    for p, pb in ((150.0, 200.0), (87.5, 287.0), (300.0, 250.0)):
        assert O.active_saving(p, pb, 0.0) == pytest.approx(1 - p / pb, rel=1e-15)
        assert O.active_saving(pb, pb, 30.0) == 0.0
        assert O.active_saving(4 * p, 4 * pb, 4 * 30.0) == O.active_saving(p, pb, 30.0)
    with pytest.raises(ValueError):
        O.active_saving(150.0, 100.0, 100.0)
    with pytest.raises(ValueError):
        O.active_saving(90.0, 200.0, 100.0)


def test_active_savings_job_hand_example():
    """DESIGN.md A29 on a two-trace job, derived by hand in exact rationals: E = [100, 300] J, T = [1, 2] s;
    baseline E_b = [150, 400] J, T_b = [1, 1.5] s; 50 W idle.  Mean powers 400/3 and 220 W; active energies
    400 - 150 = 250 J and 550 - 125 = 425 J."""
    from fractions import Fraction as F
    P, Pb, Ea, Eab = F(400, 3), F(220), F(250), F(425)
    want = (float((Pb - P) / (Pb - 50)), float(1 - Ea / Eab), float(1 - (Ea * 3) / (Eab * F(5, 2))))
    got = O.active_savings_job([100, 300], [1, 2], [150, 400], [1, 1.5], 50.0)
    assert got == pytest.approx(want, rel=1e-14)
    # with no idle power the active savings are the plain job-level power / energy / EDP savings
    got0 = O.active_savings_job([100, 300], [1, 2], [150, 400], [1, 1.5], 0.0)
    assert got0 == pytest.approx((float(1 - P / Pb), float(1 - F(400, 550)), float(1 - F(400 * 3) / F(550 * 5, 2))),
                                 rel=1e-14)


# --------------------------------------------------------------------------- NEXT-3: open-loop observation

def test_open_loop_step_hand_derived():
    """A30 (open loop, recorded throughput observed as is) on a hand-stepped rising edge: D = [2]x4 + [15]x8,
    defaults (k = 1, theta = +-1 GB/s/s, C = 10), bw_max = 22 GB/s (B_lo = 8), w = 0.5.  A = D, so the only
    tune flag is the edge at t = 4 (d = 13 GB/s over 0.1 s > 1): Increase -> f_max from t = 5, then Hold.
    No tick is throttled: T = 12 * 0.1 s; E_pkg = 200 W * 0.7 s + 116 W * 0.5 s = 198 J; E = 198 + 87 * 1.2.
    (Closed loop, A14, sees the throttled jump 2 -> 8 at f_min and then 8 -> 15: two flags, a dilated tick.)"""
    D = np.array([2.0] * 4 + [15.0] * 8, np.float32)
    r, codes = O.replay(D, 0.5, O.Policy(), O.Model(bw_max_gbps=22.0, observe=1), codes=True)
    assert (r["tune_events"], r["transitions"], r["n_hi"], r["n_thr"], r["lock_ticks"]) == (1, 1, 7, 0, 0)
    assert [int(c & 1) for c in codes] == [0] * 4 + [1] * 8
    assert r["T"] == pytest.approx(1.2, rel=1e-12) and r["E_pkg"] == pytest.approx(198.0, rel=1e-12)
    assert r["E"] == pytest.approx(198.0 + 87.0 * 1.2, rel=1e-12)
    rc, _ = O.replay(D, 0.5, O.Policy(), O.Model(bw_max_gbps=22.0), codes=True)
    assert (rc["tune_events"], rc["transitions"], rc["n_thr"]) == (2, 1, 1)


def test_open_loop_equals_closed_loop_below_b_lo():
    """A30 vs A14: when no sample exceeds B_lo no tick can be throttled at either level, so A = D in both
    modes and every record is identical, for every policy kind."""
    rng = np.random.default_rng(30)
    D = rng.uniform(0.0, 7.0, 3000).astype(np.float32)   # B_lo = 7.27 at the default model
    for pol in (O.Policy(), O.Policy(deriv_ticks=3, tune_log_capacity=5, high_freq_threshold=0.4),
                O.Policy(kind=O.TDP_DEFAULT, tdp_w=217.0), O.Policy(kind=O.STATIC_MIN)):
        a, _ = O.replay(D, 0.7, pol, O.Model(), codes=True)
        b, _ = O.replay(D, 0.7, pol, O.Model(observe=1), codes=True)
        for f in ("n_hi", "n_thr", "transitions", "tune_events", "lock_ticks", "digest", "T", "E"):
            assert a[f] == b[f], f


def test_open_loop_flags_depend_on_the_trace_only():
    """A30: with A = D the Alg. 1 signal, hence every tune flag, is a function of the trace and of (k, theta)
    alone -- the same for policies that differ only in C and theta_hf (whose levels differ); the closed loop
    has no such property on a trace that crosses B_lo (A14)."""
    rng = np.random.default_rng(31)
    D = np.repeat(rng.uniform(0.5, 19.0, 400), rng.integers(1, 6, 400))[:1500].astype(np.float32)
    pa, pb = O.Policy(tune_log_capacity=10, high_freq_threshold=0.6), O.Policy(tune_log_capacity=4, high_freq_threshold=0.5)
    _, ca = O.replay(D, 0.6, pa, O.Model(observe=1), codes=True)
    _, cb = O.replay(D, 0.6, pb, O.Model(observe=1), codes=True)
    assert np.array_equal(ca & 0x34, cb & 0x34)            # flag bit and signal bits
    assert not np.array_equal(ca & 0x81, cb & 0x81)        # while the levels do differ


# --------------------------------------------------------------------------- NEXT-3: byte counters

def test_counters_spec_examples():
    """counts 1e9 -> 2e9 over 0.1 s is 1e10 B/s (10 GB/s); equal counts are 0 B/s; a counter
    reset to 0 -> "sample discarded, no governor round": the interval yields no round at all -- the
    trace's rounds are its valid intervals in time order, padded with 0 after n_valid (A31) -- and the baseline
    re-arms, so the next interval is measured from the reset value."""
    counts = np.array([1_000_000_000, 2_000_000_000, 2_000_000_000, 0, 500_000_000], np.uint64)
    thr, nv, discarded = O.counters_to_throughput(counts, period=0.1)
    assert thr[:, 0].tolist() == [10.0, 0.0, 5.0, 0.0] and nv.tolist() == [3] and discarded == 1
    # leading resets: no round before the first valid interval (no made-up 0 GB/s sample)
    thr, nv, discarded = O.counters_to_throughput(np.array([5, 3, 1, 4_000_000_001], np.uint64), period=0.5)
    assert thr[:, 0].tolist() == [np.float32(8.0), 0.0, 0.0] and nv.tolist() == [1] and discarded == 2
    # columns are independent: each trace keeps its own rounds
    two = np.array([[0, 0], [10**9, 5], [2 * 10**9, 2], [3 * 10**9, 10**9 + 2]], np.uint64)
    thr, nv, discarded = O.counters_to_throughput(two, period=1.0)
    assert nv.tolist() == [3, 2] and discarded == 1
    assert thr[:, 0].tolist() == [1.0, 1.0, 1.0] and thr[:, 1].tolist() == [np.float32(5e-9), 1.0, 0.0]


def test_counters_timestamps_and_rounding():
    """Per-row timestamps give the difference quotient over the actual intervals; a non-increasing timestamp
    is an error; each value is the fp64 quotient rounded once to fp32 (checked against exact
    rationals)."""
    from fractions import Fraction as F
    rng = np.random.default_rng(32)
    n = 50
    steps = rng.integers(0, 3_000_000_000, (n, 3)).astype(np.uint64)
    counts = np.cumsum(steps, axis=0, dtype=np.uint64)
    times = np.cumsum(rng.uniform(0.05, 0.2, n))
    thr, nv, resets = O.counters_to_throughput(counts, times=times)
    assert resets == 0 and nv.tolist() == [n - 1] * 3
    for i in (0, 17, 48):
        for j in range(3):
            q = F(int(counts[i + 1, j] - counts[i, j])) / F(float(times[i + 1] - times[i])) / F(10**9)
            assert abs(F(float(thr[i, j])) - q) <= q * F(1, 2**23)    # within half an fp32 ulp (+ fp64 rounding)
    with pytest.raises(ValueError):
        O.counters_to_throughput(counts, times=np.r_[times[:10], times[9], times[11:]])


# --------------------------------------------------------------------------- NEXT-1: wall-clock rounds (A32)

B_LO = float(np.float32(20.0 * (0.8 / 2.2)))


def test_wallclock_spec_examples():
    """SPEC.md:356-360 (A32): at f_min with demand = 2 x B_lo and compute weight 0 an entry's work takes two
    governor rounds; with demand <= B_lo, or compute weight 1, one round.  Static-min over n entries:
    2n rounds and T = 2n * Delta (resp. n, n * Delta); E = (P_lo + P_gpu) * T."""
    n = 37
    pol = O.Policy(kind=O.STATIC_MIN)
    r, c = O.replay_wallclock(np.full(n, 2 * B_LO, np.float32), 0.0, pol, codes=True)
    assert r["n_rounds"] == 2 * n and r["n_thr"] == 2 * n and r["T"] == pytest.approx(2 * n * 0.1, rel=1e-14)
    assert r["E"] == pytest.approx((116.0 + 87.0) * 2 * n * 0.1, rel=1e-14)
    for D, w in ((np.full(n, B_LO, np.float32), 0.0), (np.full(n, 2 * B_LO, np.float32), 1.0)):
        r, _ = O.replay_wallclock(D, w, pol)
        assert r["n_rounds"] == n and r["T"] == pytest.approx(n * 0.1, rel=1e-14)
    # static max is never throttled: one entry per round, T = T_base (A2)
    D = np.random.default_rng(32).uniform(0, 20, 500).astype(np.float32)
    r, _ = O.replay_wallclock(D, 0.3, O.Policy(kind=O.STATIC_MAX))
    assert r["n_rounds"] == 500 and r["n_thr"] == 0 and r["T"] == pytest.approx(r["T_base"], rel=1e-14)


def test_wallclock_static_time_conservation():
    """A32 at a fixed level: the rounds' used time adds up to the sum of the entries' dilations, closed
    form T = Delta * sum_j (w + (1 - w) D_j / min(D_j, B_lo)) for throttled entries (1 otherwise), and the
    number of rounds is ceil(T / Delta) (every round but the last is whole)."""
    rng = np.random.default_rng(33)
    D = rng.uniform(0, 20, 2000).astype(np.float32)
    w = 0.35
    r, _ = O.replay_wallclock(D, w, O.Policy(kind=O.STATIC_MIN))
    d = D.astype(np.float64)
    dil = np.where(d > B_LO, float(np.float32(w)) + (1 - float(np.float32(w))) * d / B_LO, 1.0)
    assert r["T"] == pytest.approx(0.1 * math.fsum(dil), rel=1e-12)
    assert r["n_rounds"] == math.ceil(math.fsum(dil) - 1e-9)


def test_wallclock_equals_entry_replay_when_unthrottled():
    """A32 reduces to the per-entry replay (A14) when no round can be throttled (every D <= B_lo): one
    entry per round, identical codes, counts, digest, T and E, for every policy kind."""
    rng = np.random.default_rng(34)
    D = rng.uniform(0.0, 7.0, 3000).astype(np.float32)
    for pol in (O.Policy(), O.Policy(deriv_ticks=3, tune_log_capacity=5, high_freq_threshold=0.4),
                O.Policy(kind=O.TDP_DEFAULT, tdp_w=217.0), O.Policy(kind=O.STATIC_MAX)):
        a, ca = O.replay(D, 0.7, pol, codes=True)
        b, cb = O.replay_wallclock(D, 0.7, pol, codes=True)
        assert b["n_rounds"] == len(D) and np.array_equal(ca, cb)
        for f in ("n_hi", "n_thr", "transitions", "tune_events", "lock_ticks", "digest", "T", "E", "E_pkg"):
            assert a[f] == b[f], f


@pytest.mark.parametrize("seed,w,kind,observe", [(40, 0.0, "magus", 0), (41, 0.5, "magus", 0), (42, 0.9, "magus", 0),
                                                  (43, 0.3, "tdp", 0), (44, 0.2, "magus", 1), (45, 0.0, "static_min", 0)])
def test_wallclock_bruteforce(seed, w, kind, observe):
    """A32 against the independent brute force (tests/_bruteforce.py): exact rational time accounting,
    full-prefix Alg. 1 / Alg. 2.  Piecewise-constant traces crossing B_lo (so entries span rounds, levels
    change mid-entry, and the lock engages)."""
    rng = np.random.default_rng(seed)
    D = np.repeat(rng.uniform(0.5, 19.5, 60), rng.integers(3, 15, 60))[:300].astype(np.float32)
    k, C, hf = 2, 6, 0.5
    pk = {"magus": O.MAGUS, "tdp": O.TDP_DEFAULT, "static_min": O.STATIC_MIN}[kind]
    pol = O.Policy(kind=pk, deriv_ticks=k, tune_log_capacity=C, high_freq_threshold=hf, tdp_w=217.0)
    r, codes = O.replay_wallclock(D, w, pol, O.Model(observe=observe), codes=True)
    rows, tot = BF.replay_wallclock_prefix(D, w, k, 1.0, -1.0, C, hf, kind=kind, tdp=217.0, observe=observe)
    assert r["n_rounds"] == len(rows)
    assert np.array_equal(codes, BF.rows_to_codes(rows))
    for f in ("T", "E", "E_pkg"):
        assert r[f] == pytest.approx(tot[f], rel=1e-12), f
    if kind == "magus" and observe == 0:
        assert r["n_thr"] > 0 and r["n_rounds"] > len(D) and r["lock_ticks"] > 0 and r["transitions"] > 5


# --------------------------------------------------------------------------- K14: platform model (SPEC simsys)

def test_bandwidth_linear_spec_examples():
    """K14: Linear bandwidth_at(f_max) = bw_max; bw_max = 2e10, f_max = 2.2 GHz,
    f = 0.8 GHz -> 2e10 * 0.8/2.2 ~ 7.27e9.  A wrong ratio (f_min/f, f_max/f) fails the second value."""
    m = O.Model(bw_max_gbps=20.0)
    assert O.bandwidth_at(2.2, m) == 20.0
    assert O.bandwidth_at(0.8, m) == pytest.approx(7.2727272727, rel=1e-10)


def test_bandwidth_saturating_spec_example_and_hand_values():
    """K14: Saturating bw_max * min(1, (f/f_max)/knee).
    - S:338: knee 0.5 at f = 0.6 f_max -> bw_max (above the knee the bandwidth saturates);
    - hand value below the knee: knee 0.5, f = 0.8, f_max = 2.2, bw_max = 20 -> 20 * (0.8/2.2)/0.5
      = 14.5454...; a `ratio * knee` slip gives 3.64, a missing min() gives > bw_max above the knee;
    - exactly at the knee (f = knee * f_max) -> bw_max; knee = 1 is the Linear model;
    - non-decreasing in f, equal to bw_max at f_max (SPEC.md:317 invariants)."""
    m = O.Model(bw_max_gbps=20.0, bw_shape=1, bw_knee=0.5)
    assert O.bandwidth_at(0.6 * 2.2, m) == 20.0
    assert O.bandwidth_at(0.8, m) == pytest.approx(20.0 * (0.8 / 2.2) / 0.5, rel=1e-15)
    assert O.bandwidth_at(0.8, m) == pytest.approx(14.545454545454545, rel=1e-12)
    assert O.bandwidth_at(1.1, m) == 20.0            # f / f_max = 0.5 = knee
    assert O.bandwidth_at(2.0, m) == 20.0
    m1 = O.Model(bw_max_gbps=20.0, bw_shape=1, bw_knee=1.0)
    lin = O.Model(bw_max_gbps=20.0)
    fs = np.linspace(0.8, 2.2, 57)
    for f in fs:
        assert O.bandwidth_at(f, m1) == O.bandwidth_at(f, lin)
    for knee in (0.25, 0.5, 0.9):
        mk = O.Model(bw_max_gbps=20.0, bw_shape=1, bw_knee=knee)
        vals = [O.bandwidth_at(f, mk) for f in fs]
        assert all(b >= a for a, b in zip(vals, vals[1:]))
        assert vals[-1] == 20.0
        assert vals[0] == pytest.approx(20.0 * min(1.0, (0.8 / 2.2) / knee), rel=1e-15)


def test_uncore_power_spec_examples_and_exponent():
    """K14: p_min + (p_max - p_min) ((f - f_min)/(f_max - f_min))^e.
    Endpoints give exactly p_uncore_min / p_uncore_max for every exponent (the replay only
    ever evaluates the endpoints, A19); exponent 1 at the midpoint is the arithmetic mean;
    hand values for e = 2 (a quarter of the way up at the midpoint) and e = 3.  Package power adds
    p_pkg_idle + p_core_active: 60 + 40 + 16 = 116 W and 200 W with the default model."""
    for e in (1.0, 1.7, 2.0, 3.0):
        m = O.Model(p_exponent=e)
        assert O.uncore_power_at(0.8, m) == 16.0
        assert O.uncore_power_at(2.2, m) == 100.0
    assert O.uncore_power_at(1.5, O.Model(p_exponent=1.0)) == pytest.approx(58.0, rel=1e-14)
    assert O.uncore_power_at(1.5, O.Model(p_exponent=2.0)) == pytest.approx(16.0 + 84.0 / 4, rel=1e-14)
    assert O.uncore_power_at(1.15, O.Model(p_exponent=3.0)) == pytest.approx(16.0 + 84.0 / 64, rel=1e-13)
    assert O.pkg_power_at(0.8, O.Model()) == 116.0 and O.pkg_power_at(2.2, O.Model()) == 200.0


def test_saturating_model_in_the_replay_closed_form():
    """K14: the closed loop of the replay with the Saturating model.  With knee 0.5, B_lo =
    fl32(20 * (0.8/2.2)/0.5) = fl32(14.5454...).  STATIC_MIN on a constant demand D = 16 > B_lo is
    throttled every tick: T = N Delta (w + (1 - w) D / B_lo) (A16), E_pkg = P_lo T; on
    D = 12 < B_lo (but above the Linear B_lo 7.27) nothing is throttled, so the saturating B_lo, not the
    Linear one, is in the loop.  MAGUS on a 12 -> 16 step at f_min sees A rise only to B_lo."""
    m = O.Model(bw_shape=1, bw_knee=0.5)
    b_lo = float(np.float32(20.0 * ((0.8 / 2.2) / 0.5)))   # operand order of A26
    n, w = 200, float(np.float32(0.3))   # compute_weight is an fp32 input
    r, codes = O.replay(np.full(n, 16.0, np.float32), w, O.Policy(kind=O.STATIC_MIN), m, codes=True)
    assert r["n_thr"] == n
    assert r["T"] == pytest.approx(n * 0.1 * (w + (1 - w) * 16.0 / b_lo), rel=1e-12)
    assert r["E_pkg"] == pytest.approx(116.0 * r["T"], rel=1e-12)
    r, _ = O.replay(np.full(n, 12.0, np.float32), w, O.Policy(kind=O.STATIC_MIN), m)
    assert r["n_thr"] == 0 and r["T"] == pytest.approx(n * 0.1, rel=1e-12)
    r_lin, _ = O.replay(np.full(n, 12.0, np.float32), w, O.Policy(kind=O.STATIC_MIN), O.Model())
    assert r_lin["n_thr"] == n
    # MAGUS at f_min on 12 then 16: the observed step is 12 -> B_lo (a rise of 2.55 GB/s in one tick > 1
    # GB/s/s * 0.1 s), so Alg. 1 returns +1 and the governor goes to f_max on the step tick
    D = np.r_[np.full(50, 12.0), np.full(50, 16.0)].astype(np.float32)
    r, codes = O.replay(D, w, O.Policy(), m, codes=True)
    assert codes[49] & 1 == 0 and codes[50] & 1 == 1 and (codes[50] >> 4) & 3 == 1
    assert r["n_thr"] == 1
