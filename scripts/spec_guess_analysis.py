#!/usr/bin/env python
"""Analysis (CPU, oracle-based): how often a speculative segment's guessed warm-up start lands on the wrong entry
state, per trace class and policy, for the segment plan of a config.  Compares guess rules.  Not a test.

The true entry state at a segment start comes from the oracle's per-tick codes (level, tune flags, the observed
A values); the speculative one from a plain Python re-run of the warm-up window from the guessed level."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2502_03796_b200.configs import CONFIGS  # noqa: E402

B_LO = float(np.float32(20.0 * (0.8 / 2.2)))


def thresholds(p):
    L = p["deriv_ticks"] * 0.1
    return p["inc_threshold"] * L, p["dec_threshold"] * L   # approximate d* (analysis only)


def warm(D, t0, t1, f, p):
    """Python MAGUS ticks over [t0, t1) from level f with empty ring / log; returns (f, log tuple, ring tuple)."""
    k, C = p["deriv_ticks"], p["tune_log_capacity"]
    s_min = next(s for s in range(C + 2) if s > C or s / C >= p["high_freq_threshold"])
    dinc, ddec = thresholds(p)
    ring, log = collections.deque(), collections.deque()
    for t in range(t0, t1):
        a = float(min(D[t], B_LO)) if f == 0 else float(D[t])
        ring.append(a)
        sig = 0
        if len(ring) > k:
            d = ring[-1] - ring[0]
            ring.popleft()
            sig = 1 if d > dinc else (-1 if d < ddec else 0)
            log.append(1 if sig else 0)
            if len(log) > C:
                log.popleft()
        hf = len(log) == C and sum(log) >= s_min
        f = 1 if (hf or sig == 1) else (0 if sig == -1 else f)
    return f, tuple(log), tuple(ring)


def true_entry(D, codes, t, p):
    k, C = p["deriv_ticks"], p["tune_log_capacity"]
    f = int(codes[t] >> 7) & 1                    # level in effect at tick t
    flags = [int(c >> 2) & 1 for c, r in zip(codes[:t], range(t)) if (c >> 1) & 1][-C:]
    lv = [(int(c) >> 7) & 1 for c in codes[t - k:t]]
    ring = tuple(float(D[i]) if lv[n] else float(min(D[i], B_LO)) for n, i in enumerate(range(t - k, t)))
    return f, tuple(flags), ring


def guess_old(D, tau, first_low, first_high, p, s_min):
    hi = D[tau] > B_LO and first_low < tau
    sticky = p["deriv_ticks"] >= s_min
    return 1 if (hi or (sticky and first_low < tau and first_high < tau)) else 0


def guess_new(D, tau, first_low, first_high, p, s_min):
    k = p["deriv_ticks"]
    high = lambda t: t >= 0 and D[t] > B_LO
    now = high(tau)
    stable = all(high(tau - i) for i in range(1, 9))
    vis = any(high(tau - i) != high(tau - i - k) for i in range(0, 9))
    toggling = any(not high(tau - i) for i in range(1, 9)) and any(high(tau - i) for i in range(1, 9))
    hi = now and ((not high(tau - k)) or (first_low < tau and stable))
    sticky = k >= s_min
    return 1 if (hi or (sticky and first_low < tau and first_high < tau and (vis or not toggling))) else 0


def main():
    ci = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    per_class = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    S = int(sys.argv[3]) if len(sys.argv) > 3 else 18
    W = int(sys.argv[4]) if len(sys.argv) > 4 else 32
    c = CONFIGS[ci]
    ns = c["n_samples"]
    L = (ns // S) // 32 * 32
    pols = [p for p in c["policies"] if p["kind"] == 0]
    ncls = 5 if c["class_mix"] == 1 else (3 if c["class_mix"] == 0 else 11)
    ids = [j for j in range(ncls * per_class)]
    desc = O.GenDesc(seed=c["seed"], n_traces=max(ids) + 1, n_samples=ns, class_mix=c["class_mix"])
    wrong = collections.Counter()
    total = collections.Counter()
    for j in ids:
        D, w = O.gen_trace(desc, j)
        lows = [t for t in range(0, ns, 256) if D[t] <= B_LO]
        highs = [t for t in range(0, ns, 256) if D[t] > B_LO]
        fl = lows[0] if lows else 1 << 30
        fh = highs[0] if highs else 1 << 30
        for pi, p in enumerate(pols):
            C = p["tune_log_capacity"]
            s_min = next(s for s in range(C + 2) if s > C or s / C >= p["high_freq_threshold"])
            _, codes = O.replay(D, float(w), O.Policy(**p), codes=True)
            for s in range(1, S):
                t = s * L
                tau = t - W
                te = true_entry(D, codes, t, p)
                for name, g in (("old", guess_old), ("new", guess_new)):
                    f0 = g(D, tau, fl, fh, p, s_min)
                    se = warm(D, tau, t, f0, p)
                    key = (name, j % ncls, p["deriv_ticks"])
                    total[key] += 1
                    wrong[key] += se != te
    for name in ("old", "new"):
        print(name, "wrong entries by (class, k):",
              {k[1:]: f"{wrong[k]}/{total[k]}" for k in sorted(total) if k[0] == name and wrong[k]})
        print(name, "total wrong", sum(v for k, v in wrong.items() if k[0] == name), "of",
              sum(v for k, v in total.items() if k[0] == name))


if __name__ == "__main__":
    main()
