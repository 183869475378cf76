"""Diagnostic (GPU box only): config 3's traces under a one-k sweep (64 points, all k = KK) -- one launch group, one
kernel image per SM -- timed with 16 / 8 / 4 traces per wide-kernel CTA (MAGUS_WIDE_TPC).
usage: python scripts/wide1_probe.py KK"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2502_03796_b200 import magus as M  # noqa: E402
from paper_2502_03796_b200.configs import CONFIGS, pol  # noqa: E402

kk = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = CONFIGS[3]
n, ns = cfg["n_traces"], cfg["n_samples"]
tr = torch.empty((ns, n), dtype=torch.float32, device="cuda")
w = torch.empty(n, dtype=torch.float32, device="cuda")
M.gen_traces(cfg["seed"], n, ns, cfg["class_mix"], tr, w, trace_stride=n)
pols = [M.Policy(**pol(deriv_ticks=kk, high_freq_threshold=hf, inc_threshold=th, dec_threshold=-th))
        for hf in (0.4, 0.5, 0.6, 0.7) for th in (0.25, 0.5, 0.75, 1.0, 1.5, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12)]
for w1 in ("16", "8", "4"):
    os.environ["MAGUS_WIDE_TPC"] = w1
    R = M.Replay(n, ns, pols, M.Model(), trace_stride=n)
    for _ in range(2):
        R.run(tr, w)
        R.results()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        R.run(tr, w)
    e1.record()
    torch.cuda.synchronize()
    print(f"k={kk} MAGUS_WIDE_TPC={w1}: {e0.elapsed_time(e1) / 5:.3f} ms per run, geometry {R.geometry()}", flush=True)
    del R
