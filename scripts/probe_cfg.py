"""Diagnostic: time one config's replay at a list of forced segment counts (GPU box only).

usage: python scripts/probe_cfg.py <config> [S ...]     (S = 0: the library's own choice)
Prints one line per S: step ms, per-kernel CUDA-event times, segments, mismatches, fix-up rounds.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MAGUS_NO_REPLAN", "1")

import torch  # noqa: E402

from paper_2502_03796_b200 import magus as M  # noqa: E402
from paper_2502_03796_b200.configs import CONFIGS  # noqa: E402


def main():
    ci = int(sys.argv[1])
    segs = [int(x) for x in sys.argv[2:]] or [0]
    cfg = CONFIGS[ci]
    n = cfg.get("per_gpu_traces", cfg["n_traces"])
    ns = cfg["n_samples"]
    stride = (n + 3) // 4 * 4
    dev = torch.device("cuda", 0)
    tr = torch.empty((ns, stride), dtype=torch.float32, device=dev)
    w = torch.empty(n, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)
    M.gen_traces(cfg["seed"], n, ns, cfg["class_mix"], tr, w, trace_stride=stride, stream=stream)
    pols = [M.Policy(**d) for d in cfg["policies"]]
    for S in segs:
        R = M.Replay(n, ns, pols, M.Model(), trace_stride=stride, flags=M.F_TIMING | M.F_TIMING_DETAIL,
                     tuning_segments=S)
        for _ in range(3):
            R.run(tr, w, stream)
            res = R.results()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 10
        e0.record(stream)
        for _ in range(K):
            R.run(tr, w, stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / K
        ts = R.timing_summary(K)
        res = R.results()
        g = R.geometry()
        del R
        # the same plan without per-kernel timing events (every kernel edge programmatic)
        R2 = M.Replay(n, ns, pols, M.Model(), trace_stride=stride, tuning_segments=S)
        for _ in range(3):
            R2.run(tr, w, stream)
            R2.results()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(K):
            R2.run(tr, w, stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms2 = e0.elapsed_time(e1) / K
        del R2
        print(f"cfg{ci} S_req={S} S={res.n_segments} W={res.warmup_ticks} ms={ms:.4f} ms_notiming={ms2:.4f} "
              f"mism={res.n_mismatched_segments} rounds={res.fixup_rounds} "
              + " ".join(f"{k}={v:.4f}" for k, v in ts.items()) + f" geo={g}", flush=True)
        time.sleep(0.2)


if __name__ == "__main__":
    main()
