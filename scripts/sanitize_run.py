"""Small replays that cover every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck).  GPU box only.  usage: compute-sanitizer --tool <t> python scripts/sanitize_run.py

Covers: the generator, the pre-pass, the one-warp solo replay kernel (MAGUS k <= 3, TMA/mbarrier ring; the L stage and
variant 2), the fused one-warp MAGUS + TDP kernel (12- and 16-CTA builds), the two-warp combined MAGUS + TDP kernel
(shared ring, empty barriers), the unsegmented wide kernel (8-warp CTAs; P, L and D stages, per-warp fp64 scratch), the
multi-warp replay kernel (shared tiles: several policy warps, TDP / STATIC_MIN / k >= 4 / 64-bit logs), the
fix-up mark + split / lockstep / per-thread walks, the totals and chunk-sum kernels, the decision re-simulation,
the wall-clock kernels, the counter ingest -- direct launches and the captured CUDA graph.  Each run is checked
against the oracle (so a sanitizer run is also a parity run)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_03796_b200 import magus as M  # noqa: E402
from paper_2502_03796_b200.configs import CONFIGS, pol, sweep64, STATIC_MAX, STATIC_MIN, TDP_DEFAULT  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests import _parity as PA  # noqa: E402


def gen(seed, n, ns, mix):
    stride = (n + 3) // 4 * 4
    tr = torch.empty((ns, stride), dtype=torch.float32, device="cuda")
    w = torch.empty(n, dtype=torch.float32, device="cuda")
    M.gen_traces(seed, n, ns, mix, tr, w, trace_stride=stride)
    return tr, w, stride


def case(name, seed, n, ns, mix, pols, segments, flags=0, stream=False, model=None):
    tr, w, stride = gen(seed, n, ns, mix)
    st = torch.cuda.Stream() if stream else None
    with M.Replay(n, ns, PA.gpu_policies(pols), model or M.Model(), trace_stride=stride,
                  flags=flags | M.F_PER_TRACE_STATS | M.F_DUMP_DECISIONS, dump_first_trace=0, dump_n_traces=min(n, 3),
                  tuning_segments=segments) as R:
        R.run(tr, w, st)
        res = R.results()
        geo = R.geometry()
    torch.cuda.synchronize()
    if flags & M.F_WALLCLOCK:
        rec, _ = PA.oracle_wallclock(tr.cpu().numpy(), w.cpu().numpy(), pols, n, O.Model())
    else:
        om = O.Model(observe=model.observe) if model is not None else O.Model()
        rec, _, _ = O.replay_batch(tr.cpu().numpy()[:, :n], w.cpu().numpy(), PA.oracle_policies(pols), om)
    PA.compare_records(res.per_trace, rec, name)
    print(f"{name}: ok  segments={res.n_segments} mismatched={res.n_mismatched_segments} geometry={geo}", flush=True)


def main():
    cfg2, cfg5 = CONFIGS[2]["policies"], CONFIGS[5]["policies"]
    c1 = CONFIGS[1]
    case("cfg1", c1["seed"], 1, 4000, c1["class_mix"], c1["policies"], 0)
    case("cfg2-small solo segmented", 2, 260, 6000, 0, cfg2, 6)
    case("cfg2-small graph", 2, 260, 6000, 0, cfg2, 6, stream=True)
    case("cfg5-small solo+tdp, walks", 5, 257, 6000, 2, cfg5 + sweep64()[40:42], 7)
    case("cfg3-small shared tiles", 3, 64, 3000, 1, sweep64()[::5] + [pol(kind=STATIC_MAX)], 5)
    case("cfg5 fused MAGUS + TDP kernel (one warp), walks", 5, 257, 6000, 2, cfg5, 7)
    case("fused kernel, k = 2, asymmetric thresholds", 5, 257, 6000, 2,
         [pol(deriv_ticks=2, inc_threshold=0.7, dec_threshold=-1.3), pol(kind=TDP_DEFAULT, tdp_w=217.0)], 7)
    os.environ["MAGUS_FUSED_CTAS"] = "16"
    case("fused kernel, 16-CTA build", 5, 257, 6000, 2, cfg5, 7)
    os.environ.pop("MAGUS_FUSED_CTAS")
    os.environ["MAGUS_COMBO"] = "1"
    case("cfg5 combined two-warp MAGUS + TDP kernel, walks", 5, 257, 6000, 2, cfg5, 7)
    os.environ.pop("MAGUS_COMBO")
    os.environ["MAGUS_FUSE"] = "0"
    case("cfg5 separate MAGUS solo + TDP solo launches", 5, 257, 6000, 2, cfg5, 7)
    os.environ.pop("MAGUS_FUSE")
    case("solo L stage, asymmetric thresholds", 2, 260, 6000, 0,
         [pol(inc_threshold=0.8, dec_threshold=-1.1), pol(kind=STATIC_MAX)], 6)
    os.environ["MAGUS_SOLO_BAL"] = "2"
    case("solo stage variant 2", 2, 260, 6000, 0, cfg2, 6)
    os.environ.pop("MAGUS_SOLO_BAL")
    os.environ["MAGUS_WIDE"] = "1"
    case("cfg3-small unsegmented wide plan (P stage)", 3, 40, 3000, 1, sweep64() + [pol(kind=STATIC_MAX)], 0)
    os.environ["MAGUS_WIDE_L"] = "1"
    case("wide plan, L stage", 3, 40, 3000, 1, sweep64(), 0)
    os.environ["MAGUS_WIDE_L"] = "0"
    case("wide plan, D stage", 3, 40, 3000, 1, sweep64(), 0)
    os.environ.pop("MAGUS_WIDE_L")
    case("wide plan, asymmetric thresholds (P stage)", 3, 40, 3000, 1,
         [pol(deriv_ticks=k, inc_threshold=0.6, dec_threshold=-1.7) for k in (1, 3, 8)], 0)
    os.environ["MAGUS_WIDE_NC"] = "2"
    case("wide plan, two chains per thread", 3, 40, 3000, 1, sweep64(), 0)
    os.environ.pop("MAGUS_WIDE_NC")
    os.environ.pop("MAGUS_WIDE")
    case("k>=4, 64-bit logs, static min", 9, 131, 3000, 1,
         [pol(deriv_ticks=9, tune_log_capacity=10), pol(deriv_ticks=4, tune_log_capacity=40),
          pol(kind=STATIC_MIN), pol(kind=TDP_DEFAULT, tdp_w=217.0)], 5)
    os.environ["MAGUS_WALK_SPLIT"] = "0"
    case("lockstep walk", 5, 200, 6000, 2, cfg5 + sweep64()[40:42], 7)
    os.environ["MAGUS_WALK_LOCKSTEP"] = "0"
    case("per-thread walk", 5, 200, 6000, 2, cfg5 + sweep64()[40:42], 7)
    os.environ.pop("MAGUS_WALK_SPLIT")
    os.environ.pop("MAGUS_WALK_LOCKSTEP")
    case("open loop: O stage + closed-form fix-up", 2, 260, 6000, 0, cfg2, 9, model=M.Model(observe=1))
    case("open loop: two MAGUS groups, asymmetric thresholds", 3, 131, 3000, 1,
         [pol(deriv_ticks=3, inc_threshold=0.6, dec_threshold=-1.4), pol(deriv_ticks=1, tune_log_capacity=20)], 7,
         model=M.Model(observe=1))
    case("wall-clock rounds", 5, 96, 1500, 2, cfg5, 0, flags=M.F_WALLCLOCK)
    case("nccl exchange (world 1)", 2, 130, 3000, 0, cfg2, 4, flags=M.F_NCCL, stream=True)
    # NEXT-3 counter ingest
    rng = np.random.default_rng(1)
    counts = np.cumsum(rng.integers(0, 1_000_000_000, (300, 132)).astype(np.uint64), axis=0, dtype=np.uint64)
    tr = torch.empty((299, 132), dtype=torch.float32, device="cuda")
    counts[150:, 7] -= counts[150, 7]   # a reset
    M.counters_to_trace(torch.from_numpy(counts.view(np.int64)).cuda(), tr, 130, period_s=0.1)
    torch.cuda.synchronize()
    print("ingest: ok", flush=True)


if __name__ == "__main__":
    main()
