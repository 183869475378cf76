"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.  -m gpu.

Bars (north_star): per-tick cmd / tune-flag bits, counts and 64-bit digests
bit-exact; T, E, E_pkg, EDP and the savings within 1e-9 relative; generator bytes bit-exact.
"""
import io
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import _parity as PA
from paper_2502_03796_b200.configs import CONFIGS, pol, sweep64, STATIC_MAX, STATIC_MIN, TDP_DEFAULT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def M():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2502_03796_b200 import magus
    return magus


def gpu_gen(M, seed, n_traces, n_samples, mix, stride=None, offset=0, amp=0.002):
    stride = stride or ((n_traces + 3) // 4 * 4)
    tr = torch.empty((n_samples, stride), dtype=torch.float32, device="cuda")
    w = torch.empty(max(1, n_traces), dtype=torch.float32, device="cuda")
    M.gen_traces(seed, n_traces, n_samples, mix, tr, w, trace_stride=stride, global_trace_offset=offset,
                 noise_amp=amp)
    torch.cuda.synchronize()
    return tr, w


def run_gpu(M, tr, w, policies, n_traces, n_samples, stride, flags=None, segments=0, warmup=0, offset=0,
            dump=(0, 0), model=None):
    flags = (M.F_PER_TRACE_STATS | M.F_DUMP_WORDS) if flags is None else flags
    if dump[1]:
        flags |= M.F_DUMP_DECISIONS
    with M.Replay(n_traces, n_samples, PA.gpu_policies(policies), model or M.Model(), trace_stride=stride,
                  global_trace_offset=offset, flags=flags, dump_first_trace=dump[0], dump_n_traces=dump[1],
                  tuning_segments=segments, tuning_warmup=warmup) as R:
        R.run(tr, w)
        res = R.results()
        res.geometry = R.geometry()
    return res


def oracle_run(tr_host, w_host, policies, n_traces, model=None):
    rec, codes, _ = O.replay_batch(tr_host[:, :n_traces], w_host[:n_traces], PA.oracle_policies(policies),
                                   model or O.Model(), codes=True)
    return rec, codes


# ------------------------------------------------------------------------------------- generator

@pytest.mark.parametrize("mix,n,ns,stride,offset", [(0, 300, 3000, 304, 0), (1, 130, 2100, 132, 7),
                                                    (2, 77, 4000, 80, 1000), (3, 1, 10000, 4, 0)])
def test_generator_bytes_match_oracle(M, mix, n, ns, stride, offset):
    """a11: the CUDA generator writes exactly the oracle generator's bytes (counter-based recipe)."""
    tr, w = gpu_gen(M, 42 + mix, n, ns, mix, stride, offset)
    otr, ow = O.gen_traces(O.GenDesc(seed=42 + mix, n_traces=n, n_samples=ns, class_mix=mix, trace_stride=stride,
                                     global_trace_offset=offset))
    assert np.array_equal(tr.cpu().numpy().view(np.uint32), otr.view(np.uint32))
    assert np.array_equal(w.cpu().numpy()[:n].view(np.uint32), ow.view(np.uint32))


# ------------------------------------------------------------------------------------- config 1

def test_cfg1_every_tick(M):
    """cfg 1 (1 trace x 10,000, default policy): every per-tick code byte, every 32-tick cmd/flag word
    from the replay kernel, and the record, against the oracle."""
    c = CONFIGS[1]
    tr, w = gpu_gen(M, c["seed"], 1, c["n_samples"], c["class_mix"], c["stride"])
    res = run_gpu(M, tr, w, c["policies"], 1, c["n_samples"], c["stride"], dump=(0, 1))
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), c["policies"], 1)
    assert np.array_equal(res.decisions, codes)
    assert np.array_equal(res.words, PA.pack_words(codes))
    PA.compare_records(res.per_trace, rec, "cfg1")


# ------------------------------------------------------------------------------------- small configs

SMALL = {
    "cfg2-small": dict(seed=2, n=300, ns=20_000, mix=0, policies=CONFIGS[2]["policies"]),
    "cfg3-small": dict(seed=3, n=64, ns=4_000, mix=1, policies=CONFIGS[3]["policies"]),
    "cfg5-small": dict(seed=5, n=257, ns=8_000, mix=2, policies=CONFIGS[5]["policies"]),
    "mixed-kinds": dict(seed=9, n=131, ns=5_003, mix=1,
                        policies=[pol(), pol(kind=STATIC_MIN), pol(kind=TDP_DEFAULT, tdp_w=217.0),
                                  pol(kind=STATIC_MAX), pol(deriv_ticks=3, tune_log_capacity=4,
                                                            high_freq_threshold=0.75)]),
}


@pytest.mark.parametrize("segments", [0, 1, 7])
@pytest.mark.parametrize("name", list(SMALL))
def test_small_configs(M, name, segments):
    """Several tiles, a ragged trace tail, a ragged final block; automatic, none and forced time
    segmentation (exercises the speculative segments and the exact fix-up)."""
    s = SMALL[name]
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    res = run_gpu(M, tr, w, s["policies"], s["n"], s["ns"], stride, segments=segments,
                  dump=(max(0, s["n"] - 5), 5))
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), s["policies"], s["n"])
    PA.compare_records(res.per_trace, rec, name)
    assert np.array_equal(res.words, PA.pack_words(codes))
    assert np.array_equal(res.decisions, codes[:, s["n"] - 5:, :])
    PA.compare_totals(res.totals, rec)
    edp = PA.oracle_totals(rec)[:, 3]
    assert res.totals[res.argmin_policy, 3] <= edp.min() * (1 + 1e-9)
    if segments == 7:
        assert res.n_segments == 7


@pytest.mark.parametrize("segments", [0, 5])
@pytest.mark.parametrize("name", ["mixed-kinds", "cfg5-small", "cfg2-small"])
def test_saturating_bandwidth_model(M, name, segments):
    """SPEC.md:330-338 Saturating bandwidth (bw_shape = 1) with knee 0.5: B_lo = fl32(20 (0.8/2.2)/0.5)
    = 14.545 GB/s instead of the Linear 7.27, so the throttle threshold, the closed-loop observation and
    the energy epilogue all run on the saturating value; records, words and a code dump against the
    oracle's replay under the same model."""
    s = SMALL[name]
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    th = M.derive_thresholds(M.Policy(), M.Model(bw_shape=1, bw_knee=0.5))
    assert th["B_lo"] == np.float32(20.0 * ((0.8 / 2.2) / 0.5)) != np.float32(20.0 * (0.8 / 2.2))
    res = run_gpu(M, tr, w, s["policies"], s["n"], s["ns"], stride, segments=segments, dump=(0, 4),
                  model=M.Model(bw_shape=1, bw_knee=0.5))
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), s["policies"], s["n"],
                            model=O.Model(bw_shape=1, bw_knee=0.5))
    PA.compare_records(res.per_trace, rec, f"saturating {name}")
    assert np.array_equal(res.words, PA.pack_words(codes))
    assert np.array_equal(res.decisions, codes[:, :4, :])
    PA.compare_totals(res.totals, rec)
    lin, _ = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), s["policies"], s["n"])
    assert not np.array_equal(lin["n_thr"], rec["n_thr"])   # the model changed what the loop saw


@pytest.mark.parametrize("k,C,hf", [(1, 1, 1.0), (2, 10, 0.6), (5, 7, 0.5), (8, 10, 0.4), (9, 10, 0.6),
                                    (16, 33, 0.6), (33, 64, 0.5), (64, 64, 0.9), (4, 64, 0.3), (7, 40, 0.6),
                                    (1, 32, 0.6), (3, 33, 0.6)])
def test_window_and_log_sizes(M, k, C, hf):
    """Every k in the register-ring specialisations and the generic ring, C up to 64 (64-bit log),
    with forced segmentation so warm-up lengths scale with k + C."""
    n, ns = 140, 6000
    tr, w = gpu_gen(M, 100 + k, n, ns, 1, 140)
    pols = [pol(deriv_ticks=k, tune_log_capacity=C, high_freq_threshold=hf, inc_threshold=0.5, dec_threshold=-0.5)]
    res = run_gpu(M, tr, w, pols, n, ns, 140, segments=5)
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, n)
    PA.compare_records(res.per_trace, rec, f"k={k} C={C}")
    assert np.array_equal(res.words, PA.pack_words(codes))


@pytest.mark.parametrize("model", ["closed", "open"])
@pytest.mark.parametrize("bal", ["24", "20"])
@pytest.mark.parametrize("C,k,th", [(7, 1, 0.5), (8, 1, 0.5), (8, 3, 1.0), (9, 2, 0.5), (10, 1, 1.0), (16, 3, 0.5),
                                    (23, 2, 1.0), (24, 1, 0.5), (24, 3, 1.0), (25, 1, 0.5)])
def test_batched_flag_log(M, C, k, th, bal, model, monkeypatch):
    """The solo L stage (closed loop) and O stage (open loop, A30) with the tune-flag log shifted once per stage
    (BAL 24 / 25 and 34 / 35, 8 <= C <= 24) at both ends of its C range and just outside it
    (C = 7, 25: the per-tick shift), with the |d| (symmetric) and the two-compare tests, against the oracle;
    MAGUS_SOLO_BAL=20 forces the per-tick shift."""
    monkeypatch.setenv("MAGUS_SOLO_BAL", bal)
    n, ns = 140, 6000
    tr, w = gpu_gen(M, 300 + C + k, n, ns, 1, 140)
    pols = [pol(deriv_ticks=k, tune_log_capacity=C, high_freq_threshold=0.6, inc_threshold=th,
                dec_threshold=-th if k != 2 else -0.75 * th)]
    gm = (M.Model(observe=1), O.Model(observe=1)) if model == "open" else (M.Model(), O.Model())
    res = run_gpu(M, tr, w, pols, n, ns, 140, segments=5, model=gm[0])
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, n, model=gm[1])
    PA.compare_records(res.per_trace, rec, f"batched log C={C} k={k} BAL {bal} {model}")
    assert np.array_equal(res.words, PA.pack_words(codes))


WIDE_CASES = {
    # config 3's 64-point sweep (k in {1, 2, 4, 8}: four launch groups of 16 points) + static max
    "cfg3-small": (SMALL["cfg3-small"]["policies"], 64, 4_000, 1),
    # every register-ring k, logs up to C = 28, 3 points per group (13 idle lanes per 16), a ragged trace count
    # and a ragged last block
    "k1-8": ([pol(deriv_ticks=k, tune_log_capacity=C, high_freq_threshold=hf, inc_threshold=th, dec_threshold=-th)
              for k in range(1, 9) for (C, hf, th) in ((10, 0.6, 1.0), (28, 0.5, 0.5), (3, 0.7, 2.0))],
             133, 5_003, 3),
    # shorter than the warm-up of the longest log (k + C - 1 > n_samples) and a single partial block
    "short": ([pol(deriv_ticks=k, tune_log_capacity=28) for k in (1, 4, 8)] + [pol(kind=STATIC_MAX)], 21, 33, 1),
}


@pytest.mark.parametrize("model", ["linear", "saturating", "open-loop"])
@pytest.mark.parametrize("name", list(WIDE_CASES))
def test_wide_unsegmented_plan(M, name, model, monkeypatch):
    """The unsegmented one-chain-per-lane plan (magus_replay_wide_kernel), forced with
    MAGUS_WIDE=1: records, every tick's cmd / tune-flag word, a decision dump and the totals against the oracle,
    under the Linear and Saturating bandwidth models and the open-loop observation (A30)."""
    monkeypatch.setenv("MAGUS_WIDE", "1")
    pols, n, ns, mix = WIDE_CASES[name]
    stride = (n + 3) // 4 * 4
    tr, w = gpu_gen(M, 31 + n, n, ns, mix, stride)
    gm = dict(linear=(M.Model(), O.Model()), saturating=(M.Model(bw_shape=1, bw_knee=0.5), O.Model(bw_shape=1, bw_knee=0.5)),
              **{"open-loop": (M.Model(observe=1), O.Model(observe=1))})[model]
    res = run_gpu(M, tr, w, pols, n, ns, stride, dump=(n - 3, 3), model=gm[0])
    geo = res.geometry
    assert geo["wide_groups"] == geo["launch_groups"] and res.n_segments == 1, geo
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, n, model=gm[1])
    PA.compare_records(res.per_trace, rec, f"wide {name} {model}")
    assert np.array_equal(res.words, PA.pack_words(codes))
    assert np.array_equal(res.decisions, codes[:, n - 3:, :])
    PA.compare_totals(res.totals, rec)
    edp = PA.oracle_totals(rec)[:, 3]
    assert res.totals[res.argmin_policy, 3] <= edp.min() * (1 + 1e-9)


def test_wide_plan_choice(M, monkeypatch):
    """The automatic plan picks the unsegmented kernel for config 3's sweep (65,536 chains) and the segmented
    solo kernel for config 2 (4,096 chains); MAGUS_WIDE=0 turns it off."""
    for ci, want in ((3, 4), (2, 0)):
        c = CONFIGS[ci]
        with M.Replay(c["n_traces"], c["n_samples"], PA.gpu_policies(c["policies"]), trace_stride=c["stride"]) as R:
            g = R.geometry()
        assert g["wide_groups"] == want, (ci, g)
        assert (g["n_segments"] == 1) == (want > 0), (ci, g)
    monkeypatch.setenv("MAGUS_WIDE", "0")
    c = CONFIGS[3]
    with M.Replay(c["n_traces"], c["n_samples"], PA.gpu_policies(c["policies"]), trace_stride=c["stride"]) as R:
        assert R.geometry()["wide_groups"] == 0


@pytest.mark.parametrize("combo", ["1", "0"])
@pytest.mark.parametrize("n_tdp", [1, 2])
def test_combo_kernel_reads_each_tile_once(M, combo, n_tdp, monkeypatch):
    """Config 5's policy mix (MAGUS + static max + TDP_DEFAULT baselines) runs as ONE two-warp kernel sharing the
    TMA tiles (magus_replay_combo_kernel: MAGUS warp + TDP warp) -- and, with MAGUS_COMBO=0, as two launches; both
    equal the oracle (records, every word, a decision dump, totals), with forced segmentation so the fix-up walks
    run after the combined replay."""
    monkeypatch.setenv("MAGUS_COMBO", combo)
    monkeypatch.setenv("MAGUS_NO_TDP_CLOSED", "1")   # replay the 270 W policy too (it never leaves f_max)
    s = SMALL["cfg5-small"]
    pols = s["policies"][:2 + n_tdp]
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    res = run_gpu(M, tr, w, pols, s["n"], s["ns"], stride, segments=9, dump=(s["n"] - 4, 4))
    geo = res.geometry
    assert geo["launch_groups"] == 2
    assert (geo["threads_per_cta"] == 64) == (combo == "1"), geo
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, s["n"])
    PA.compare_records(res.per_trace, rec, f"combo={combo} tdp={n_tdp}")
    assert np.array_equal(res.words, PA.pack_words(codes))
    assert np.array_equal(res.decisions, codes[:, s["n"] - 4:, :])
    PA.compare_totals(res.totals, rec)


@pytest.mark.parametrize("fuse,ctas,bal", [("1", "12", "24"), ("1", "12", "20"), ("1", "16", "24"), ("0", "12", "24")])
@pytest.mark.parametrize("k", [1, 3])
@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("segments", [9, 1])
def test_fused_magus_tdp_kernel(M, fuse, ctas, bal, k, sym, segments, monkeypatch):
    """One MAGUS policy next to one replayed TDP_DEFAULT baseline (config 5's replayed pair) runs as ONE warp per (tile
    group, segment) stepping both chain kinds over the same samples (magus_replay_fused_kernel, MAGUS_FUSE=1, built
    for 12 or 16 CTAs per SM) -- one replay launch instead of two; with MAGUS_FUSE=0 as two launches.  Both equal the
    oracle (records, every word, a decision dump, totals), with k in {1, 3}, symmetric (the |d| test) and asymmetric
    thresholds, and forced segmentation (speculative entries, fix-up walks after the fused replay) or none; bal 24 =
    the batched tune-flag log (C = 10), 20 = the per-tick shift."""
    monkeypatch.setenv("MAGUS_SOLO_BAL", bal)
    monkeypatch.setenv("MAGUS_FUSE", fuse)
    monkeypatch.setenv("MAGUS_FUSED_CTAS", ctas)
    s = SMALL["cfg5-small"]
    th = dict(inc_threshold=1.0, dec_threshold=-1.0) if sym else dict(inc_threshold=0.7, dec_threshold=-1.3)
    pols = [pol(deriv_ticks=k, **th), pol(kind=TDP_DEFAULT, tdp_w=217.0)]
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    res = run_gpu(M, tr, w, pols, s["n"], s["ns"], stride, segments=segments, dump=(s["n"] - 4, 4))
    geo = res.geometry
    assert geo["launch_groups"] == 2
    monkeypatch.setenv("MAGUS_FUSE", "0")
    with M.Replay(s["n"], s["ns"], PA.gpu_policies(pols), trace_stride=stride, tuning_segments=segments) as R2:
        unfused = R2.geometry()
    assert geo["kernels_per_run"] == unfused["kernels_per_run"] - (1 if fuse == "1" else 0), (geo, unfused)
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, s["n"])
    PA.compare_records(res.per_trace, rec, f"fuse={fuse} ctas={ctas} bal={bal} k={k} sym={sym} S={segments}")
    assert np.array_equal(res.words, PA.pack_words(codes))
    assert np.array_equal(res.decisions, codes[:, s["n"] - 4:, :])
    PA.compare_totals(res.totals, rec)


@pytest.mark.parametrize("ns", [8011, 97])
@pytest.mark.parametrize("kind", ["fused", "open-fast"])
def test_ragged_lengths_new_paths(M, ns, kind, monkeypatch):
    """The fused MAGUS + TDP kernel and the open-loop fast path on a trace length that is not a multiple of 32 (the
    ragged last block runs the per-tick paths: the TDP tick from the level bit of its cmd word, the event word of the
    O stage) and on a trace shorter than the warm-up, with forced segmentation where the length allows."""
    monkeypatch.setenv("MAGUS_FUSE", "1")
    monkeypatch.setenv("MAGUS_OPEN_FAST", "1")
    s = SMALL["cfg5-small"]
    pols = [pol(), pol(kind=TDP_DEFAULT, tdp_w=217.0)] if kind == "fused" else [pol(deriv_ticks=2), pol(kind=STATIC_MAX)]
    mk = dict(observe=1) if kind == "open-fast" else {}
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], ns, s["mix"], stride)
    res = run_gpu(M, tr, w, pols, s["n"], ns, stride, segments=7 if ns > 2000 else 0, dump=(s["n"] - 4, 4),
                  model=M.Model(**mk))
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, s["n"], model=O.Model(**mk))
    PA.compare_records(res.per_trace, rec, f"{kind} ns={ns}")
    assert np.array_equal(res.words, PA.pack_words(codes))
    assert np.array_equal(res.decisions, codes[:, s["n"] - 4:, :])
    PA.compare_totals(res.totals, rec)


@pytest.mark.parametrize("model", ["saturating", "open-loop", "short-period"])
def test_fused_kernel_models(M, model, monkeypatch):
    """The fused MAGUS + TDP kernel under the other observation / bandwidth models: Saturating bandwidth (B_lo from the
    knee), open loop (A = D, no tick throttled: the throttle bound is +inf) and a shorter sample period -- records,
    every word and totals equal the oracle's, with forced segmentation."""
    monkeypatch.setenv("MAGUS_FUSE", "1")
    s = SMALL["cfg5-small"]
    mk = dict(saturating=dict(bw_shape=1, bw_knee=0.5), **{"open-loop": dict(observe=1)},
              **{"short-period": dict(sample_period_s=0.05)})[model]
    pols = [pol(), pol(kind=TDP_DEFAULT, tdp_w=217.0)]
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    res = run_gpu(M, tr, w, pols, s["n"], s["ns"], stride, segments=7, model=M.Model(**mk))
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, s["n"], model=O.Model(**mk))
    PA.compare_records(res.per_trace, rec, f"fused {model}")
    assert np.array_equal(res.words, PA.pack_words(codes))
    PA.compare_totals(res.totals, rec)


def _random_case(seed):
    """A seeded random run: sizes (ragged, sometimes tiny), policies of every kind with random parameters (MAGUS k, C
    up to 64, thresholds; TDP budgets around the model's power range), a random model (Linear / Saturating, closed or
    open loop, sample period) and edge samples injected into generated traces (0, -0.0, B_lo and its neighbours,
    bw_max, the largest fp32 below it, the smallest subnormal, 1e-30)."""
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 3, 17, 64, 131, 257]))
    ns = int(rng.choice([1, 31, 33, 640, 2049, 5003]))
    pols = []
    for _ in range(int(rng.integers(1, 7))):
        kind = int(rng.choice([0, 0, 0, 1, 2, 3]))
        if kind == 0:
            pols.append(pol(deriv_ticks=int(rng.choice([1, 2, 3, 4, 5, 8, 9, 16, 33, 64])),
                            tune_log_capacity=int(rng.choice([1, 2, 4, 10, 20, 28, 29, 40, 64])),
                            high_freq_threshold=float(rng.choice([0.05, 0.3, 0.5, 0.6, 0.75, 1.0])),
                            inc_threshold=float(rng.uniform(0.05, 5.0)), dec_threshold=-float(rng.uniform(0.05, 5.0))))
        elif kind == 3:
            pols.append(pol(kind=TDP_DEFAULT, tdp_w=float(rng.uniform(150.0, 300.0)),
                            tdp_margin=float(rng.uniform(0.01, 0.2))))
        else:
            pols.append(pol(kind=STATIC_MAX if kind == 1 else STATIC_MIN))
    mk = dict(sample_period_s=float(rng.choice([0.05, 0.1, 0.25])), observe=int(rng.integers(0, 2)))
    if rng.integers(0, 2):
        mk.update(bw_shape=1, bw_knee=float(rng.choice([0.3, 0.5, 1.0])))
    segments = int(rng.choice([0, 0, 1, 3, 9]))
    wide = bool(rng.integers(0, 2))
    return n, ns, int(rng.integers(0, 4)), pols, mk, segments, wide, rng


N_RANDOM = int(os.environ.get("MAGUS_RANDOM_SEEDS", "24"))   # more seeds for a longer sweep (evidence runs)


@pytest.mark.parametrize("seed", list(range(N_RANDOM)))
def test_randomized_runs_with_edge_samples(M, seed, monkeypatch):
    """Seeded random runs (_random_case) against the oracle: every record, every tick's cmd / tune-flag word and the
    totals.  Sizes, policies, models, plans (segmented / unsegmented / forced segment counts) all vary."""
    n, ns, mix, pols, mk, segments, wide, rng = _random_case(seed)
    if wide:
        monkeypatch.setenv("MAGUS_WIDE", "1")
    stride = (n + 3) // 4 * 4
    tr, w = gpu_gen(M, 500 + seed, n, ns, mix, stride)
    h = tr.cpu().numpy()
    B_lo = np.float32(M.derive_thresholds(M.Policy(), M.Model(**mk))["B_lo"])
    edges = np.array([0.0, -0.0, B_lo, np.nextafter(B_lo, np.float32(0)), np.nextafter(B_lo, np.float32(30)), 20.0,
                      np.nextafter(np.float32(20.0), np.float32(0)), np.float32(1.4e-45), 1e-30], dtype=np.float32)
    edges = edges[edges <= np.float32(20.0)]   # valid samples only (A17): B_lo's upper neighbour may exceed bw_max
    n_edge = max(1, (ns * n) // 50)
    rows, cols = rng.integers(0, ns, n_edge), rng.integers(0, n, n_edge)
    h[rows, cols] = edges[rng.integers(0, len(edges), n_edge)]
    tr.copy_(torch.from_numpy(h))
    res = run_gpu(M, tr, w, pols, n, ns, stride, segments=segments, model=M.Model(**mk))
    rec, codes = oracle_run(h, w.cpu().numpy(), pols, n, model=O.Model(**mk))
    label = f"seed {seed}: n={n} ns={ns} segments={segments} wide={wide} model={mk} policies={pols}"
    PA.compare_records(res.per_trace, rec, label)
    assert np.array_equal(res.words, PA.pack_words(codes)), label
    PA.compare_totals(res.totals, rec)


@pytest.mark.parametrize("seed", list(range(max(8, N_RANDOM // 2))))
def test_randomized_round2_paths(M, seed, monkeypatch):
    """Seeded random runs aimed at the round-2 paths, with edge samples: one MAGUS policy next to one TDP_DEFAULT
    policy (the fused kernel), open-loop MAGUS-only runs (the O stage and the closed-form fix-up), and MAGUS sweeps
    in the unsegmented plan (the wide P stage with balanced CTAs) -- random k <= 8, C <= 27, thresholds (symmetric
    or not), TDP budgets, sizes and segment counts; records, every word and the totals against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    path = ["fused", "open", "wide"][seed % 3]
    n = int(rng.choice([37, 129, 300, 517]))
    ns = int(rng.choice([700, 2049, 4096, 5003]))
    def mpol(kmax):
        th = float(rng.uniform(0.05, 4.0))
        sym = bool(rng.integers(0, 2))
        return pol(deriv_ticks=int(rng.integers(1, kmax + 1)), tune_log_capacity=int(rng.choice([2, 5, 10, 16, 27])),
                   high_freq_threshold=float(rng.choice([0.3, 0.5, 0.6, 0.8])), inc_threshold=th,
                   dec_threshold=-th if sym else -float(rng.uniform(0.05, 4.0)))
    mk = {}
    segments = int(rng.choice([1, 3, 9, 17]))
    if path == "fused":
        pols = [mpol(3), pol(kind=TDP_DEFAULT, tdp_w=float(rng.uniform(205.0, 260.0)))]
        monkeypatch.setenv("MAGUS_FUSE", "1")
    elif path == "open":
        pols = [mpol(3)] + ([mpol(3)] if rng.integers(0, 2) else []) + [pol(kind=STATIC_MAX)]
        mk = dict(observe=1)
    else:
        pols = [mpol(8) for _ in range(int(rng.integers(4, 20)))]
        monkeypatch.setenv("MAGUS_WIDE", "1")
        segments = 0
    stride = (n + 3) // 4 * 4
    tr, w = gpu_gen(M, 900 + seed, n, ns, int(rng.integers(0, 4)), stride)
    h = tr.cpu().numpy()
    B_lo = np.float32(M.derive_thresholds(M.Policy(), M.Model(**mk))["B_lo"])
    edges = np.array([0.0, -0.0, B_lo, np.nextafter(B_lo, np.float32(0)), np.nextafter(B_lo, np.float32(30)), 20.0,
                      np.nextafter(np.float32(20.0), np.float32(0)), np.float32(1.4e-45), 1e-30], dtype=np.float32)
    edges = edges[edges <= np.float32(20.0)]
    n_edge = max(1, (ns * n) // 60)
    rows, cols = rng.integers(0, ns, n_edge), rng.integers(0, n, n_edge)
    h[rows, cols] = edges[rng.integers(0, len(edges), n_edge)]
    tr.copy_(torch.from_numpy(h))
    res = run_gpu(M, tr, w, pols, n, ns, stride, segments=segments, model=M.Model(**mk))
    rec, codes = oracle_run(h, w.cpu().numpy(), pols, n, model=O.Model(**mk))
    label = f"seed {seed} ({path}): n={n} ns={ns} segments={segments} model={mk} policies={pols}"
    PA.compare_records(res.per_trace, rec, label)
    assert np.array_equal(res.words, PA.pack_words(codes)), label
    PA.compare_totals(res.totals, rec)


@pytest.mark.parametrize("closed", ["0", "1"])
def test_tdp_never_low_closed_form(M, closed, monkeypatch):
    """A TDP_DEFAULT policy whose budget is never reached at f_max (config 5's 270 W: a*_hi = 113 GB/s > bw_max) is
    STATIC_MAX in closed form; replayed (MAGUS_NO_TDP_CLOSED=1) or not, every record, word, code and total equals
    the oracle's replay of the TDP policy, and the 217 W policy (which does reach its budget) is replayed."""
    monkeypatch.setenv("MAGUS_NO_TDP_CLOSED", "0" if closed == "1" else "1")
    s = SMALL["cfg5-small"]
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    th = M.derive_thresholds(M.Policy(kind=TDP_DEFAULT, tdp_w=270.0), M.Model())
    assert th["astar_hi"] > 20.0
    res = run_gpu(M, tr, w, s["policies"], s["n"], s["ns"], stride, dump=(0, 5))
    assert res.geometry["lane_policies"] == (2 if closed == "1" else 3), res.geometry
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), s["policies"], s["n"])
    PA.compare_records(res.per_trace, rec, f"tdp closed={closed}")
    assert np.array_equal(res.words, PA.pack_words(codes))
    assert np.array_equal(res.decisions, codes[:, :5, :])
    PA.compare_totals(res.totals, rec)


@pytest.mark.parametrize("name,segments", [("cfg5-small", 7), ("mixed-kinds", 5), ("cfg3-small", 0)])
def test_decision_dump_decoded_from_replay_words(M, name, segments, monkeypatch):
    """The decision dump (magus_decode_kernel: codes decoded from the replay kernels' own cmd / tune-flag words, the
    fix-up walk's rewritten blocks included) equals the independent re-simulation from t = 0 (magus_resim_kernel,
    MAGUS_DUMP_RESIM=1) and the oracle's codes byte for byte, for every dumped trace, policy and tick."""
    s = dict(SMALL[name])
    if name == "cfg5-small":
        s["policies"] = s["policies"] + sweep64()[40:42]   # lock-sticky points: speculative entries do mismatch
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    dump = (0, s["n"])
    dec = run_gpu(M, tr, w, s["policies"], s["n"], s["ns"], stride, flags=M.F_PER_TRACE_STATS, segments=segments,
                  dump=dump)
    monkeypatch.setenv("MAGUS_DUMP_RESIM", "1")
    rsm = run_gpu(M, tr, w, s["policies"], s["n"], s["ns"], stride, flags=M.F_PER_TRACE_STATS, segments=segments,
                  dump=dump)
    _, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), s["policies"], s["n"])
    assert np.array_equal(dec.decisions, rsm.decisions)
    assert np.array_equal(dec.decisions, codes)
    print(f"{name}: {dec.n_mismatched_segments} wrong speculative entries walked (their blocks' words rewritten)")


@pytest.mark.parametrize("case", ["long-trace", "long-trace-wide", "many-traces"])
def test_large_shapes(M, case, monkeypatch):
    """Maximum-size edges: traces longer than 2^24 ticks (the solo kernel's fp32 per-segment counters force a second
    segment even when one is requested; the wide kernel flushes its counters per 32-tick block) and a very wide
    trace set (300,000 traces: grid sizes, the per-trace records).  Records, totals (and the words of the long
    traces) against the oracle."""
    if case.startswith("long-trace"):
        n, ns, segments = 4, (1 << 24) + 101, (1 if case == "long-trace" else 0)
        pols = CONFIGS[2]["policies"] if case == "long-trace" else [pol(deriv_ticks=k) for k in (1, 2, 4, 8)]
        if case == "long-trace-wide":
            monkeypatch.setenv("MAGUS_WIDE", "1")
        flags = M.F_PER_TRACE_STATS | M.F_DUMP_WORDS
    else:
        n, ns, segments, pols, flags = 300_000, 64, 0, CONFIGS[5]["policies"], M.F_PER_TRACE_STATS
    stride = (n + 3) // 4 * 4
    tr, w = gpu_gen(M, 77, n, ns, 1, stride)
    res = run_gpu(M, tr, w, pols, n, ns, stride, flags=flags, segments=segments)
    if case == "long-trace":
        assert res.n_segments == 2, res.geometry    # the 2^24-tick cap
    if case == "long-trace-wide":
        assert res.geometry["wide_groups"] > 0 and res.n_segments == 1, res.geometry
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, n)
    PA.compare_records(res.per_trace, rec, case)
    PA.compare_totals(res.totals, rec)
    if flags & M.F_DUMP_WORDS:
        assert np.array_equal(res.words, PA.pack_words(codes))


@pytest.mark.parametrize("n,ns", [(1, 1), (1, 31), (3, 33), (5, 32), (128, 64), (129, 95), (4, 1000)])
def test_tiny_and_ragged(M, n, ns):
    stride = (n + 3) // 4 * 4
    tr, w = gpu_gen(M, 7, n, ns, 1, stride)
    pols = CONFIGS[5]["policies"]
    res = run_gpu(M, tr, w, pols, n, ns, stride)
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, n)
    PA.compare_records(res.per_trace, rec, f"{n}x{ns}")
    assert np.array_equal(res.words, PA.pack_words(codes))


def test_empty_inputs(M):
    """n_samples = 0 and n_traces = 0 are valid and give zero totals."""
    tr = torch.zeros((1, 4), device="cuda")
    w = torch.zeros(4, device="cuda")
    res = run_gpu(M, tr, w, CONFIGS[2]["policies"], 3, 0, 4)
    assert np.all(res.per_trace["T"] == 0) and np.all(res.per_trace["n_hi"] == 0)
    res = run_gpu(M, tr, w, CONFIGS[2]["policies"], 0, 100, 4)
    assert np.all(res.totals == 0)
    with M.Replay(3, 0, PA.gpu_policies(CONFIGS[2]["policies"]), trace_stride=4, flags=M.F_PER_TRACE_STATS) as R:
        R.run_host(np.zeros((0, 4), np.float32), np.full(3, 0.5, np.float32))   # the host path, no samples
        res = R.results()
    assert np.all(res.per_trace["T"] == 0) and res.totals[0, 12] == 3
    # the same in the wall-clock time model (A32): no rounds, zero records and totals
    pols = CONFIGS[5]["policies"]
    res = run_gpu(M, tr, w, pols, 3, 0, 4, flags=M.F_PER_TRACE_STATS | M.F_WALLCLOCK)
    rec, _ = PA.oracle_wallclock(np.zeros((0, 3), np.float32), np.zeros(3, np.float32), pols, 3, O.Model())
    PA.compare_records(res.per_trace, rec, "wallclock n_samples=0")
    assert np.all(res.per_trace["T"] == 0) and np.all(res.per_trace["digest"] == 0)
    res = run_gpu(M, tr, w, pols, 0, 100, 4, flags=M.F_WALLCLOCK)
    assert np.all(res.totals == 0)


def test_handwritten_trace_through_gpu(M):
    """The hand-derived worked trace ex2 (tests/golden) replayed by the CUDA path in a 4-trace tile."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_traces.json")))
    case = [c for c in g["cases"] if c["name"] == "ex2"][0]
    D = np.array(case["D"], np.float32)
    tr = torch.tensor(np.repeat(D[:, None], 4, axis=1)).cuda()
    w = torch.full((4,), 0.5, device="cuda")
    res = run_gpu(M, tr, w, [pol(tune_log_capacity=4, high_freq_threshold=0.75)], 4, len(D), 4,
                  model=M.Model(bw_max_gbps=22.0), dump=(0, 4))
    levels = "".join("H" if c >> 7 else "L" for c in res.decisions[:, 0, 0])
    assert levels == case["level"]
    assert res.per_trace["transitions"][0, 0] == case["transitions"]
    assert res.per_trace["E"][0, 0] == pytest.approx(case["E"], rel=1e-12)
    assert res.per_trace["T"][0, 0] == pytest.approx(case["T"], rel=1e-12)


def test_invalid_samples_reported(M):
    """A17: the first invalid (trace, tick) is reported as MAGUS_ERR_TRACE; -0.0 is valid."""
    n, ns = 300, 2000
    tr, w = gpu_gen(M, 3, n, ns, 0, 300)
    tr[100, 200] = -0.0
    res = run_gpu(M, tr, w, [pol()], n, ns, 300)
    assert res.status == 0
    tr[1500, 250] = float("nan")
    tr[700, 251] = -1.0
    tr[900, 250] = 25.0
    with pytest.raises(M.MagusError) as e:
        run_gpu(M, tr, w, [pol()], n, ns, 300)
    assert e.value.status == M.ERR_TRACE
    with M.Replay(n, ns, PA.gpu_policies([pol()]), trace_stride=300) as R:
        R.run(tr, w)
        r = R.results(raise_on_trace_error=False)
    assert (r.err_trace, r.err_tick) == (250, 900)


def test_config_errors(M):
    """invalid configs are rejected at create with the key named."""
    bad = [pol(deriv_ticks=0), pol(dec_threshold=0.5), pol(inc_threshold=-1.0), pol(tune_log_capacity=65),
           pol(high_freq_threshold=0.0), pol(kind=TDP_DEFAULT, tdp_margin=1.5), pol(deriv_ticks=65)]
    for b in bad:
        with pytest.raises(M.MagusError) as e:
            M.Replay(4, 10, PA.gpu_policies([b]))
        assert e.value.status == M.ERR_CONFIG
    with pytest.raises(M.MagusError) as e:
        M.Replay(4, 10, PA.gpu_policies([pol()]), M.Model(f_min_ghz=2.5))
    assert e.value.status == M.ERR_CONFIG and "f_max_ghz" in str(e.value)
    with pytest.raises(M.MagusError) as e:
        M.Replay(4, 10, PA.gpu_policies([pol()]), trace_stride=6)
    assert e.value.status == M.ERR_ALIGN


def test_determinism_and_virtual_ranks(M):
    """K13 on one GPU: two runs are bit-identical; splitting the traces into two shards (global ids)
    gives the same per-trace records and digests, and the totals agree to 1e-9."""
    n, ns = 512, 12_000
    tr, w = gpu_gen(M, 11, n, ns, 1, 512)
    pols = CONFIGS[5]["policies"]
    a = run_gpu(M, tr, w, pols, n, ns, 512)
    b = run_gpu(M, tr, w, pols, n, ns, 512)
    assert a.per_trace.tobytes() == b.per_trace.tobytes() and np.array_equal(a.totals, b.totals)
    half = n // 2
    parts = []
    for r in range(2):
        trs, ws = gpu_gen(M, 11, half, ns, 1, half, offset=r * half)
        parts.append(run_gpu(M, trs, ws, pols, half, ns, half, offset=r * half))
    joined = np.concatenate([p.per_trace for p in parts])
    for k in PA.EXACT:
        assert np.array_equal(joined[k], a.per_trace[k])
    np.testing.assert_allclose(parts[0].totals[:, :12] + parts[1].totals[:, :12], a.totals[:, :12], rtol=1e-9)


@pytest.mark.parametrize("graph", [False, True])
def test_nccl_exchange_world1_equals_local(M, graph):
    """The cross-rank exchange on one B200 (MAGUS_F_NCCL at world = 1: a one-rank NCCL communicator):
    magus_chunk_sum_kernel, then ncclAllReduce on the run's stream -- inside the captured CUDA graph on a
    non-default stream -- give the same per-policy totals (the chunks are added in the same order) and the
    same argmin as the host sum without NCCL, and both equal the oracle's totals within 1e-9."""
    s = SMALL["cfg5-small"]
    pols = s["policies"] + [pol(deriv_ticks=2, high_freq_threshold=0.4)]
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    st = torch.cuda.Stream() if graph else None
    out = {}
    for nccl in (0, 1):
        with M.Replay(s["n"], s["ns"], PA.gpu_policies(pols), trace_stride=stride,
                      flags=M.F_PER_TRACE_STATS | (M.F_NCCL if nccl else 0)) as R:
            for _ in range(2):                  # graph capture, then a replay of the captured graph
                R.run(tr, w, st)
                res = R.results()
            res.geometry = R.geometry()
        out[nccl] = res
    assert np.array_equal(out[0].totals, out[1].totals) and out[0].argmin_policy == out[1].argmin_policy
    assert out[1].geometry["kernels_per_run"] == out[0].geometry["kernels_per_run"] + 1
    assert out[0].per_trace.tobytes() == out[1].per_trace.tobytes()
    rec, _ = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, s["n"])
    PA.compare_totals(out[1].totals, rec)


def test_parameter_grid_slices(M):
    """North star "shards by trace and parameter grid" on one GPU: a 2 x 2 grid of
    virtual ranks (two trace shards x two policy slices, magus_grid_plan) run one after the other; each
    rank's per-trace records are its block of the single run's records, its totals land in its policy rows of
    the global [P][13], and the four add up to the single run's totals (argmin equal).  With the exchange on
    (MAGUS_F_NCCL, one rank), a slice that leaves global policies without an owner is refused at create by the
    cross-rank consistency check (MAGUS_ERR_CONFIG), and a full slice passes it."""
    s = SMALL["mixed-kinds"]
    pols = s["policies"]
    n, ns, P = s["n"], s["ns"], len(s["policies"])
    tr, w = gpu_gen(M, s["seed"], n, ns, s["mix"], (n + 3) // 4 * 4)
    full = run_gpu(M, tr, w, pols, n, ns, (n + 3) // 4 * 4, flags=M.F_PER_TRACE_STATS)
    acc = np.zeros_like(full.totals)
    for r in range(4):
        t0, nt, p0, npol = M.grid_plan(4, r, 2, n, P)
        trs, ws = gpu_gen(M, s["seed"], nt, ns, s["mix"], offset=t0)
        with M.Replay(nt, ns, PA.gpu_policies(pols[p0:p0 + npol]), trace_stride=(nt + 3) // 4 * 4,
                      global_trace_offset=t0, flags=M.F_PER_TRACE_STATS, n_policies_global=P,
                      policy_offset=p0) as R:
            R.run(trs, ws)
            res = R.results()
        assert res.totals.shape == full.totals.shape
        assert np.all(res.totals[:p0] == 0) and np.all(res.totals[p0 + npol:] == 0)
        assert res.per_trace.tobytes() == np.ascontiguousarray(full.per_trace[t0:t0 + nt, p0:p0 + npol]).tobytes()
        acc += res.totals
    np.testing.assert_allclose(acc, full.totals, rtol=1e-12)
    assert M.totals_argmin(acc) == full.argmin_policy
    with pytest.raises(M.MagusError) as e:
        M.Replay(n, ns, PA.gpu_policies(pols[:2]), flags=M.F_NCCL, n_policies_global=P, policy_offset=0)
    assert e.value.status == M.ERR_CONFIG and "owned by no rank" in str(e.value)
    with M.Replay(n, ns, PA.gpu_policies(pols), flags=M.F_NCCL, n_policies_global=P) as R:
        R.run(tr, w)
        res = R.results()
    np.testing.assert_allclose(res.totals, full.totals, rtol=1e-12)


def test_graph_path_matches_direct(M):
    """On a non-default stream the library replays each run as a captured CUDA graph; results equal the
    direct (stream-ordered launches) path, across graph reuse and a re-capture after a buffer change."""
    n, ns = 300, 6000
    tr, w = gpu_gen(M, 13, n, ns, 0, 300)
    pols = PA.gpu_policies(CONFIGS[5]["policies"])
    with M.Replay(n, ns, pols, trace_stride=300, flags=M.F_PER_TRACE_STATS | M.F_TIMING | M.F_TIMING_DETAIL) as R:
        R.run(tr, w)                              # default stream: direct launches
        direct = R.results()
        st = torch.cuda.Stream()
        outs = []
        for _ in range(3):                        # capture once, replay twice
            R.run(tr, w, st)
            outs.append(R.results())
        tr2 = tr.clone()
        R.run(tr2, w, st)                         # new buffer: re-capture
        outs.append(R.results())
        t = R.timing_summary(3)
    for o in outs:
        assert o.per_trace.tobytes() == direct.per_trace.tobytes() and np.array_equal(o.totals, direct.totals)
    assert t["replay_ms"] > 0 and t["run_ms"] >= t["replay_ms"]


def test_repeated_runs_reuse_scratch(M):
    """One handle, alternating inputs, graph and direct launches: every run equals the oracle.  The run
    scratch (segment-boundary counters, worklists, per-chain totals) is re-armed inside the kernels, so a
    stale word would corrupt the following run; the inputs are chosen so that speculative segment entries
    do mismatch (adversarial traces, lock-sticky sweep policies)."""
    n, ns, S = 200, 9_000, 9
    pols = CONFIGS[5]["policies"] + sweep64()[40:44]
    data = [gpu_gen(M, 21, n, ns, 2, 200), gpu_gen(M, 22, n, ns, 1, 200)]
    refs = []
    for tr, w in data:
        rec, _ = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, n)
        refs.append(rec)
    st = torch.cuda.Stream()
    with M.Replay(n, ns, PA.gpu_policies(pols), trace_stride=200, flags=M.F_PER_TRACE_STATS,
                  tuning_segments=S) as R:
        mism = 0
        for it in range(6):
            tr, w = data[it % 2]
            R.run(tr, w, st if it >= 2 else None)
            res = R.results()
            mism += res.n_mismatched_segments
            PA.compare_records(res.per_trace, refs[it % 2], f"run {it}")
            PA.compare_totals(res.totals, refs[it % 2])
    assert mism > 0, "inputs should exercise the fix-up"


def test_host_buffer_path(M):
    """magus_replay_run_host (the e2e path) gives the same results as the device path."""
    n, ns = 256, 5000
    tr, w = gpu_gen(M, 12, n, ns, 0, 256)
    dev = run_gpu(M, tr, w, CONFIGS[2]["policies"], n, ns, 256)
    th, wh = tr.cpu().pin_memory(), w.cpu().pin_memory()
    with M.Replay(n, ns, PA.gpu_policies(CONFIGS[2]["policies"]), trace_stride=256, flags=M.F_PER_TRACE_STATS) as R:
        R.run_host(th, wh)
        host = R.results()
    assert dev.per_trace.tobytes() == host.per_trace.tobytes()


# ------------------------------------------------------------------------------------- full size

def _oracle_all_traces(desc, n, policies, chunk, words_gpu=None, word_ids=None, model=None):
    """The oracle over EVERY local trace of a generated shard (its own generator, trace by trace, all host
    cores), in chunks; returns its records [n][P].  With words_gpu ([P][n][n_blocks][2] from the replay
    kernel, MAGUS_F_DUMP_WORDS), every trace in word_ids (default: all) also has its per-tick cmd and
    tune-flag bits compared with the oracle's codes; returns (records, traces whose words were compared)."""
    pols = PA.oracle_policies(policies)
    rec = np.zeros((n, len(pols)), dtype=O.RESULT_DTYPE)
    want_words = set(range(n)) if word_ids is None else set(int(j) for j in word_ids)
    n_words = 0
    for a in range(0, n, chunk):
        ids = np.arange(a, min(n, a + chunk))
        wid = [j for j in ids if j in want_words] if words_gpu is not None else []
        rest = np.setdiff1d(ids, np.array(wid, np.int64))
        if len(rest):
            r, _, _ = O.gen_replay(desc, rest, pols, model)
            rec[rest] = r
        if wid:
            wid = np.array(wid, np.int64)
            r, codes, _, _ = O.gen_replay_codes(desc, wid, pols, model)
            rec[wid] = r
            want = PA.pack_words_tpn(codes)
            got = words_gpu[:, wid]
            bad = np.argwhere(np.any(got != want, axis=-1))
            assert bad.size == 0, f"per-tick words differ at (policy, trace, block) {bad[0].tolist()}"
            n_words += len(wid)
    return rec, n_words


@pytest.mark.parametrize("cfg", [2, 5, 3])
def test_full_size_every_trace(M, cfg):
    """BASELINE.json full sizes in the bench's launch configuration (automatic segmentation): the GPU replays
    every trace; the oracle regenerates EVERY trace with its own generator and replays it under EVERY policy.
    Bit-exact: every (trace, policy) record's counts and digest, and every tick's cmd and tune-flag bit from
    the replay kernel's 32-tick words (MAGUS_F_DUMP_WORDS; cfg 3: the words of 256 traces x 65 policies, the
    records of all 1,024); 1e-9: T, E, E_pkg, EDP, the savings and the per-policy totals against the oracle's
    (math.fsum) totals.  A 64-trace decision dump (decoded from the replay kernel's words, magus_decode_kernel) is
    checked against those words and, byte for byte, against the oracle's codes."""
    c = CONFIGS[cfg]
    n, ns = c["n_traces"], c["n_samples"]
    tr, w = gpu_gen(M, c["seed"], n, ns, c["class_mix"], c["stride"])
    dump0 = n - 64
    res = run_gpu(M, tr, w, c["policies"], n, ns, c["stride"],
                  flags=M.F_PER_TRACE_STATS | M.F_DUMP_WORDS, dump=(dump0, 64))
    del tr
    desc = O.GenDesc(seed=c["seed"], n_traces=n, n_samples=ns, class_mix=c["class_mix"])
    word_ids = None if cfg != 3 else np.r_[np.arange(0, 128), np.arange(n - 128, n)]
    rec, n_words = _oracle_all_traces(desc, n, c["policies"], 32 if cfg == 3 else 256, res.words, word_ids)
    PA.compare_records(res.per_trace, rec, f"cfg{cfg}")
    PA.compare_totals(res.totals, rec)
    edp = PA.oracle_totals(rec)[:, 3]
    assert res.totals[res.argmin_policy, 3] <= edp.min() * (1 + 1e-9)
    # the decision dump's cmd / tune-flag bits are the replay kernel's own words ...
    assert np.array_equal(PA.pack_words(res.decisions), res.words[:, dump0:])
    # ... and every code byte (level, ready, flag, lock, signal, throttled) is the oracle's
    _, codes, _, _ = O.gen_replay_codes(desc, np.arange(dump0, n), PA.oracle_policies(c["policies"]))
    assert np.array_equal(res.decisions, np.transpose(codes, (2, 0, 1)))
    if cfg in (2, 5) and os.environ.get("MAGUS_SEG_BALANCE", "1") != "0":
        # the two-length segment plan is what these runs exercise: cfg 2, 17 x 1376 + 57 x 1344 ticks (16 one-warp
        # CTAs per SM); cfg 5, the fused MAGUS + TDP kernel at 12 CTAs per SM: 55 segments
        geo = res.geometry
        if cfg == 2 or os.environ.get("MAGUS_FUSE", "1") == "0":
            assert geo["n_segments"] == 74 and geo["seg_long"] == 17, geo
        else:
            assert geo["n_segments"] == 55, geo
    P = len(c["policies"])
    print(f"cfg{cfg}: compared records of {n} x {P} (trace, policy) chains, per-tick words of {n_words} x {P} "
          f"chains ({n_words * P * ns:,} ticks), codes of 64 x {P}; geometry {res.geometry}, "
          f"mismatched segments {res.n_mismatched_segments}")


def test_cfg4_shard_every_trace(M, monkeypatch):
    """cfg 4 as one rank of the 8-GPU run sees it (rank 5: global traces [40960, 49152) x 10^6 samples,
    32.8 GB), in the bench's launch configuration, and again with the solo kernel's synthetic warm-up state
    (MAGUS_SOLO_SYNTH=1): it lands the oscillating class (C4) on phase-shifted limit cycles, so speculative
    entries stay wrong through whole traces and the chain walk runs over ~10^6 ticks.  EVERY trace of the
    shard is regenerated and replayed by the oracle: counts and digests bit-exact, 1e-9 on energies and on
    the per-policy totals, both times; the per-tick words of 64 traces (both shard ends and C4 traces)
    bit-exact."""
    c = CONFIGS[4]
    n, ns, rank = c["per_gpu_traces"], c["n_samples"], 5
    off = rank * n
    tr, w = gpu_gen(M, c["seed"], n, ns, c["class_mix"], n, offset=off)
    desc = O.GenDesc(seed=c["seed"], n_traces=n, n_samples=ns, class_mix=c["class_mix"], global_trace_offset=off)
    word_ids = np.r_[np.arange(0, 24), np.arange(n - 24, n), np.arange(4, 4 * 5 * 16, 5)[:16] + 100]
    mism = []
    rec = None
    for synth in ("0", "1"):
        monkeypatch.setenv("MAGUS_SOLO_SYNTH", synth)
        flags = M.F_PER_TRACE_STATS | (M.F_DUMP_WORDS if synth == "0" else 0)
        res = run_gpu(M, tr, w, c["policies"], n, ns, n, flags=flags, offset=off)
        if rec is None:
            rec, n_words = _oracle_all_traces(desc, n, c["policies"], 512, res.words, word_ids)
            assert n_words == len(set(word_ids.tolist()))
        PA.compare_records(res.per_trace, rec, f"cfg4-shard synth={synth}")
        PA.compare_totals(res.totals, rec)
        mism.append(res.n_mismatched_segments)
        print(f"synth {synth}: compared {n} x {len(c['policies'])} records; geometry {res.geometry}, "
              f"mismatched {res.n_mismatched_segments}, walked {res.fixup_rounds}")
        del res
    if mism[1] == 0:
        pytest.fail("the synthetic warm-up state should exercise the chain walk")


def test_active_savings_from_gpu_totals(M):
    """NEXT-4: active power / energy / EDP savings of MAGUS against the static-max baseline from
    the GPU run's per-policy totals, with the paper's single-GPU (30 W) and 4-GPU (200 W) idle powers
    (P:397), equal the oracle's job-level active savings from its own per-trace records (1e-9)."""
    c = SMALL["cfg2-small"]
    tr, w = gpu_gen(M, c["seed"], c["n"], c["ns"], c["mix"])
    res = run_gpu(M, tr, w, c["policies"], c["n"], c["ns"], (c["n"] + 3) // 4 * 4, flags=M.F_PER_TRACE_STATS)
    rec, _ = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), c["policies"], c["n"])
    for p_idle in (30.0, 200.0):
        got = M.active_savings(res.totals, 0, 1, p_idle)
        want = O.active_savings_job(rec["E"][:, 0], rec["T"][:, 0], rec["E"][:, 1], rec["T"][:, 1], p_idle)
        np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("segments", [0, 5])
def test_open_loop_mode(M, segments):
    """NEXT-3 open-loop observation (magus_model.observe = 1, DESIGN A30: a recorded throughput observed as
    is, A = D, never throttled) on the mixed-kinds set: per-trace records, 32-tick words and per-tick codes
    equal the oracle's open-loop replay; no tick is throttled."""
    s = SMALL["mixed-kinds"]
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    res = run_gpu(M, tr, w, s["policies"], s["n"], s["ns"], stride, segments=segments, dump=(0, 4),
                  model=M.Model(observe=1))
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), s["policies"], s["n"], model=O.Model(observe=1))
    PA.compare_records(res.per_trace, rec, "open-loop")
    assert np.array_equal(res.words, PA.pack_words(codes))
    assert np.array_equal(res.decisions, codes[:, :4, :])
    assert int(rec["n_thr"].sum()) == 0 and int(res.per_trace["n_thr"].sum()) == 0
    PA.compare_totals(res.totals, rec)


@pytest.mark.parametrize("fast", ["1", "0"])
@pytest.mark.parametrize("case", ["cfg2", "cfg5-k2", "cfg3-k3-asym"])
@pytest.mark.parametrize("segments", [37, 5])
def test_open_loop_fast_fixup(M, fast, case, segments, monkeypatch):
    """Open loop with MAGUS solo groups only: the O stage records each segment's first event and the closed-form
    open-loop fix-up (magus_fix_openloop_kernel) corrects wrong speculative entry levels without a chain walk
    (MAGUS_OPEN_FAST=1); with MAGUS_OPEN_FAST=0 the L stage and the chain walk.  Many short segments so that many
    entries are wrong and many segments have no event at all (flat compute- / memory-bound traces) -- records, every
    word, a decision dump and totals equal the oracle's open-loop replay."""
    monkeypatch.setenv("MAGUS_OPEN_FAST", fast)
    name, pols = dict(cfg2=("cfg2-small", CONFIGS[2]["policies"]),
                      **{"cfg5-k2": ("cfg5-small", [pol(deriv_ticks=2), pol(kind=STATIC_MAX)]),
                         "cfg3-k3-asym": ("cfg3-small", [pol(deriv_ticks=3, inc_threshold=0.6, dec_threshold=-1.4),
                                                         pol(deriv_ticks=1, tune_log_capacity=20)])})[case]
    s = SMALL[name]
    stride = (s["n"] + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], s["n"], s["ns"], s["mix"], stride)
    res = run_gpu(M, tr, w, pols, s["n"], s["ns"], stride, segments=segments, dump=(s["n"] - 4, 4),
                  model=M.Model(observe=1))
    rec, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, s["n"], model=O.Model(observe=1))
    PA.compare_records(res.per_trace, rec, f"open-loop fast={fast} {case} S={segments}")
    assert np.array_equal(res.words, PA.pack_words(codes))
    assert np.array_equal(res.decisions, codes[:, s["n"] - 4:, :])
    PA.compare_totals(res.totals, rec)
    print(f"open loop {case} S={segments} fast={fast}: {res.n_mismatched_segments} wrong entries corrected")


@pytest.mark.parametrize("with_times", [False, True])
def test_counters_to_trace_and_open_loop_replay(M, with_times):
    """NEXT-3 front end: recorded byte counters (with wraps / resets, some at the start of a trace or at a
    256-row chunk boundary, a ragged column count) -> trace on the GPU equals the oracle's conversion bit for bit,
    and so do the per-trace round counts (a discarded interval yields no round, A31); the open-loop replay of the
    first min(n_valid) rounds (A30) equals the oracle's open-loop replay of its own conversion."""
    rng = np.random.default_rng(33)
    n, rows, stride = 150, 3001, 152
    steps = rng.integers(0, 1_700_000_000, (rows, stride)).astype(np.uint64)   # <= 19 GB/s over >= 0.09 s
    steps[rng.random((rows, stride)) < 0.3] //= 40                              # low phases
    counts = np.cumsum(steps, axis=0, dtype=np.uint64)
    for i, j in sorted(zip(rng.integers(1, rows, 40), rng.integers(0, n, 40))):   # counter resets, in time
        counts[i:, j] -= counts[i, j] - np.uint64(rng.integers(0, 1000))        # order (values stay >= 0)
    counts[1:, 5] -= counts[1, 5] - np.uint64(3)                                  # reset in the first interval
    counts[257:, 9] -= counts[257, 9] - np.uint64(1)                              # ... at a chunk boundary
    times = np.cumsum(rng.uniform(0.09, 0.11, rows)) if with_times else None
    want, want_nv, want_resets = O.counters_to_throughput(counts, period=0.1, times=times, n_traces=n)
    want[:, n:] = 0.0
    dc = torch.from_numpy(counts.view(np.int64)).cuda()
    dt = torch.from_numpy(times).cuda() if with_times else None
    tr = torch.empty((rows - 1, stride), dtype=torch.float32, device="cuda")
    nv, resets, bad = M.counters_to_trace(dc, tr, n, period_s=0.1, times=dt)
    assert bad == 0 and resets == want_resets > 0 and np.array_equal(nv, want_nv)
    assert want_nv.min() < rows - 1
    assert np.array_equal(tr.cpu().numpy().view(np.uint32), want.view(np.uint32))
    w = torch.full((n,), 0.7, dtype=torch.float32, device="cuda")
    pols = [pol(), pol(kind=STATIC_MAX), pol(deriv_ticks=2, tune_log_capacity=6)]
    ns = int(want_nv.min())
    res = run_gpu(M, tr[:ns], w, pols, n, ns, stride, segments=4, model=M.Model(observe=1))
    rec, _ = oracle_run(want[:ns], np.full(n, 0.7, np.float32), pols, n, model=O.Model(observe=1))
    PA.compare_records(res.per_trace, rec, "counters open loop")


def test_trace_csv_to_gpu_timeline(M, tmp_path):
    """NEXT-3 end to end: a SPEC trace CSV -> the device layout -> the replay with a decision dump -> the
    timeline CSV of the replay's own per-tick codes, byte-identical to the timeline formatted from the oracle's
    codes of the same trace (closed and open loop)."""
    from paper_2502_03796_b200 import traceio as T
    rng = np.random.default_rng(34)
    D0 = np.repeat(rng.choice([1.5, 3.0, 12.0, 16.0], 300), rng.integers(1, 9, 300))[:1200].astype(np.float32)
    path = tmp_path / "trace.csv"
    path.write_text("# period=0.1\nstep,demand_gbps,compute_weight\n" +
                    "".join(f"{t},{float(x)!r},0.6\n" for t, x in enumerate(D0)))
    D, wgt, per = T.read_trace_csv(str(path))
    assert np.array_equal(D, D0) and per == 0.1
    pols = [pol(), pol(kind=STATIC_MAX), pol(kind=TDP_DEFAULT, tdp_w=217.0)]
    tr = torch.zeros((len(D), 4), dtype=torch.float32, device="cuda")
    tr[:, 0] = torch.from_numpy(D).cuda()
    w = torch.full((1,), wgt, dtype=torch.float32, device="cuda")
    for observe in (0, 1):
        res = run_gpu(M, tr, w, pols, 1, len(D), 4, dump=(0, 1), model=M.Model(observe=observe))
        _, codes = oracle_run(tr.cpu().numpy(), w.cpu().numpy(), pols, 1, model=O.Model(observe=observe))
        got, want = io.StringIO(), io.StringIO()
        T.write_timeline(got, res.decisions, D, ["magus", "static_max", "tdp217"], 0.8, 2.2, per)
        T.write_timeline(want, codes, D, ["magus", "static_max", "tdp217"], 0.8, 2.2, per)
        assert got.getvalue() == want.getvalue()


# ------------------------------------------------------------------------------------- NEXT-1 wall clock

@pytest.mark.parametrize("roundmajor,unroll", [(0, 0), (0, 1), (1, 0)])
@pytest.mark.parametrize("name,observe", [("mixed-kinds", 0), ("cfg3-small", 0), ("cfg5-small", 0),
                                          ("mixed-kinds", 1)])
def test_wallclock_rounds(M, name, observe, roundmajor, unroll, monkeypatch):
    """NEXT-1 (MAGUS_F_WALLCLOCK, DESIGN A32): governor rounds of Delta wall time, throttled entries spanning
    several rounds.  Per-(trace, policy) records (counts and digests per round, bit-exact; T / E within 1e-9),
    the first n_samples rounds' codes of a dump window, and the totals, against the oracle's
    oracle_replay_wallclock."""
    monkeypatch.setenv("MAGUS_WALL_ROUNDMAJOR", str(roundmajor))   # entry-major kernels (default) / the A32 loop
    monkeypatch.setenv("MAGUS_WALL_UNROLL", str(unroll))           # rolled / unrolled entry blocks
    s = SMALL[name]
    n, ns = min(s["n"], 96), min(s["ns"], 4000)
    stride = (n + 3) // 4 * 4
    tr, w = gpu_gen(M, s["seed"], n, ns, s["mix"], stride)
    res = run_gpu(M, tr, w, s["policies"], n, ns, stride, flags=M.F_PER_TRACE_STATS | M.F_WALLCLOCK,
                  dump=(n - 6, 6), model=M.Model(observe=observe))
    rec, codes = PA.oracle_wallclock(tr.cpu().numpy(), w.cpu().numpy(), s["policies"], n,
                                     O.Model(observe=observe), dump=(n - 6, 6))
    PA.compare_records(res.per_trace, rec, f"wallclock {name}")
    assert np.array_equal(res.decisions, codes)
    PA.compare_totals(res.totals, rec)
    if observe == 0:
        assert rec["T"].sum() > ns * 0.1 * n * 1.001   # entries did span rounds
    if roundmajor:
        assert res.geometry["kernels_per_run"] == 3
    assert res.geometry["threads_per_cta"] == 128 and res.geometry["solo_groups"] == 0
    assert res.geometry["ctas"] == (n + 127) // 128 * res.geometry["lane_policies"]


def test_wallclock_edge_cases(M):
    """A32 edge cases: one sample, a 31/33-round ragged digest block, an all-throttled static-min trace at
    2 x B_lo with w = 0 (exactly two rounds per entry), and invalid samples still reported."""
    b_lo = float(np.float32(20.0 * (0.8 / 2.2)))
    pols = [pol(), pol(kind=STATIC_MIN), pol(kind=STATIC_MAX)]
    for ns, val in ((1, 5.0), (31, 2 * b_lo), (33, 1.0), (40, 2 * b_lo)):
        n = 4
        tr = torch.full((ns, n), val, dtype=torch.float32, device="cuda")
        w = torch.zeros(n, dtype=torch.float32, device="cuda")
        res = run_gpu(M, tr, w, pols, n, ns, n, flags=M.F_PER_TRACE_STATS | M.F_WALLCLOCK, dump=(0, 2))
        rec, codes = PA.oracle_wallclock(tr.cpu().numpy(), w.cpu().numpy(), pols, n, O.Model(), dump=(0, 2))
        PA.compare_records(res.per_trace, rec, f"edge ns={ns}")
        assert np.array_equal(res.decisions, codes)
        if val == 2 * b_lo:
            assert res.per_trace["T"][0, 1] == pytest.approx(2 * ns * 0.1, rel=1e-12)
    tr = torch.full((50, 4), 3.0, dtype=torch.float32, device="cuda")
    tr[17, 2] = float("nan")
    w = torch.zeros(4, dtype=torch.float32, device="cuda")
    with M.Replay(4, 50, PA.gpu_policies(pols), M.Model(), trace_stride=4, flags=M.F_WALLCLOCK) as R:
        R.run(tr, w)
        with pytest.raises(M.MagusError):
            R.results()


@pytest.mark.parametrize("cfg", [2, 5])
def test_wallclock_full_size_sampled(M, cfg):
    """NEXT-1 (A32) at BASELINE.json full sizes in the launch configuration `bench.py --wallclock` times
    (entry-major kernels, unrolled for these chain counts): the oracle regenerates sampled traces (both ends
    included) and replays them in wall-clock rounds; counts and digests bit-exact, T / E within 1e-9."""
    c = CONFIGS[cfg]
    n, ns = c["n_traces"], c["n_samples"]
    tr, w = gpu_gen(M, c["seed"], n, ns, c["class_mix"], c["stride"])
    res = run_gpu(M, tr, w, c["policies"], n, ns, c["stride"], flags=M.F_PER_TRACE_STATS | M.F_WALLCLOCK)
    del tr
    rng = np.random.default_rng(100 + cfg)
    ids = np.unique(np.r_[rng.choice(n, 8, replace=False), [0, n - 1]])
    desc = O.GenDesc(seed=c["seed"], n_traces=n, n_samples=ns, class_mix=c["class_mix"])
    cols = [O.gen_trace(desc, int(j)) for j in ids]            # the oracle's own generator, trace by trace
    otr = np.stack([col for col, _ in cols], axis=1)
    ow = np.array([wj for _, wj in cols], np.float32)
    rec, _ = PA.oracle_wallclock(otr, ow, c["policies"], len(ids), O.Model())
    PA.compare_records(res.per_trace[ids], rec, f"wallclock cfg{cfg}")
    np.testing.assert_allclose(res.totals, PA.oracle_totals(res.per_trace), rtol=1e-9)
    assert rec["T"].sum() > rec["T_base"].sum()   # throttled entries spanned rounds


@pytest.mark.parametrize("unroll", [0, 1])
def test_wallclock_window_and_log_sizes(M, unroll, monkeypatch):
    """NEXT-1 (A32) through every ticker the wall-clock kernels instantiate: register rings k = 3, 5, 7, the
    generic ring (k = 9, 16), the 64-bit tune log (C = 33, 64), TDP at 270 W, static min; records and codes
    against the oracle."""
    monkeypatch.setenv("MAGUS_WALL_UNROLL", str(unroll))
    n, ns = 70, 3000
    tr, w = gpu_gen(M, 77, n, ns, 1, 72)
    pols = [pol(deriv_ticks=3, tune_log_capacity=5, high_freq_threshold=0.5, inc_threshold=0.5, dec_threshold=-0.5),
            pol(deriv_ticks=5, tune_log_capacity=7), pol(deriv_ticks=7, tune_log_capacity=12),
            pol(deriv_ticks=9, tune_log_capacity=10), pol(deriv_ticks=16, tune_log_capacity=33, high_freq_threshold=0.5),
            pol(deriv_ticks=3, tune_log_capacity=64, high_freq_threshold=0.3),
            pol(kind=TDP_DEFAULT, tdp_w=270.0), pol(kind=STATIC_MIN)]
    res = run_gpu(M, tr, w, pols, n, ns, 72, flags=M.F_PER_TRACE_STATS | M.F_WALLCLOCK, dump=(0, 3))
    rec, codes = PA.oracle_wallclock(tr.cpu().numpy(), w.cpu().numpy(), pols, n, O.Model(), dump=(0, 3))
    PA.compare_records(res.per_trace, rec, "wallclock k/C")
    assert np.array_equal(res.decisions, codes)
    assert rec["lock_ticks"].sum() > 0 and rec["n_thr"].sum() > 0
