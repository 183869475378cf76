"""The five BASELINE.json configurations as concrete synthetic inputs.

Shared by tests and bench.py (the product never imports oracle/; this module only names inputs).  Holds only sizes, seeds and policy-parameter points -- none of the
method's arithmetic.
"""
from __future__ import annotations

MAGUS, STATIC_MAX, STATIC_MIN, TDP_DEFAULT = 0, 1, 2, 3

DEFAULT = dict(kind=MAGUS, deriv_ticks=1, inc_threshold=1.0, dec_threshold=-1.0, tune_log_capacity=10,
               high_freq_threshold=0.6, tdp_w=270.0, tdp_margin=0.05)


def pol(**kw):
    d = dict(DEFAULT)
    d.update(kw)
    return d


def sweep64():
    """cfg 3: k in {1,2,4,8} x theta_hf in {.4,.5,.6,.7} x theta in {.5,1,2,4}; p = 16 i_k + 4 i_hf + i_theta."""
    out = []
    for k in (1, 2, 4, 8):
        for hf in (0.4, 0.5, 0.6, 0.7):
            for th in (0.5, 1.0, 2.0, 4.0):
                out.append(pol(deriv_ticks=k, high_freq_threshold=hf, inc_threshold=th, dec_threshold=-th))
    return out


CONFIGS = {
    1: dict(name="cfg1-single-trace", seed=1, n_traces=1, n_samples=10_000, class_mix=3, stride=4,
            policies=[pol()]),
    2: dict(name="cfg2-4096x1e5-mixed", seed=2, n_traces=4096, n_samples=100_000, class_mix=0, stride=4096,
            policies=[pol(), pol(kind=STATIC_MAX)]),
    3: dict(name="cfg3-1024x1e5-sweep64", seed=3, n_traces=1024, n_samples=100_000, class_mix=1, stride=1024,
            policies=sweep64() + [pol(kind=STATIC_MAX)]),
    4: dict(name="cfg4-65536x1e6-sharded", seed=4, n_traces=65_536, n_samples=1_000_000, class_mix=1, stride=65_536,
            policies=[pol(), pol(kind=STATIC_MAX)], per_gpu_traces=8192),
    5: dict(name="cfg5-4096x1e5-adversarial", seed=5, n_traces=4096, n_samples=100_000, class_mix=2, stride=4096,
            policies=[pol(), pol(kind=STATIC_MAX), pol(kind=TDP_DEFAULT, tdp_w=270.0),
                      pol(kind=TDP_DEFAULT, tdp_w=217.0)]),
}
