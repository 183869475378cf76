"""Independent brute-force re-statement of the MAGUS loop, used to pin the oracle (K10, K12).

Test helper only.  It shares nothing with oracle/ or the product: it keeps the
*entire* observed prefix and the entire list of tune flags, and re-evaluates
Alg. 1 and Alg. 2 from those full lists
at every tick -- no FIFOs, no incremental state (SPEC.md:214 / AC3).
Energy is integrated with math.fsum (exactly rounded) instead of a running sum.
"""
import math

import numpy as np

LO, HI = 0, 1


def f32(x):
    return float(np.float32(x))


def replay_prefix(D, w, k, inc, dec, C, hf_thr, *, dt=0.1, bw_max=20.0, f_min=0.8, f_max=2.2,
                  p_idle=60.0, p_core=40.0, p_umin=16.0, p_umax=100.0, p_gpu=87.0, kind="magus",
                  tdp=270.0, margin=0.05, c_dram=0.5):
    B = {LO: f32(bw_max * (f_min / f_max)), HI: f32(bw_max * (f_max / f_max))}
    P = {LO: (p_idle + p_core) + p_umin, HI: (p_idle + p_core) + (p_umin + (p_umax - p_umin) * 1.0)}
    f = LO if kind in ("magus", "static_min") else HI
    observed, flags = [], []
    rows, taus_pkg, taus_all, taus = [], [], [], []
    for t, d in enumerate(D):
        d = f32(d)
        a = min(d, B[f])
        thr = a < d
        tau = dt * (float(w) + (1.0 - float(w)) * (d / a)) if thr else dt
        taus.append(tau)
        taus_pkg.append(P[f] * tau)
        taus_all.append((P[f] + p_gpu) * tau)
        observed.append(a)
        sig, ready, hf = 0, False, False
        if kind == "magus":
            if len(observed) >= k + 1:                      # Alg. 1 over the last k periods of the prefix
                ready = True
                deriv = (observed[-1] - observed[-1 - k]) / (k * dt)
                sig = 1 if deriv > inc else (-1 if deriv < dec else 0)
                flags.append(1 if sig != 0 else 0)
            if len(flags) >= C:                             # Alg. 2 over the last C flags of the prefix
                window = flags[-C:]
                hf = (sum(window) / len(window)) >= hf_thr
            cmd = HI if hf else (HI if sig == 1 else (LO if sig == -1 else f))
        elif kind == "tdp":
            cmd = LO if (P[f] + c_dram * a) >= (1.0 - margin) * tdp else HI
        else:
            cmd = f
        rows.append(dict(level=f, cmd=cmd, ready=ready, event=int(ready and sig != 0), hf=hf, sig=sig, thr=thr))
        f = cmd
    T = math.fsum(taus)
    return rows, dict(T=T, E_pkg=math.fsum(taus_pkg), E=math.fsum(taus_all))


def rows_to_codes(rows):
    out = []
    for r in rows:
        c = (r["cmd"] == HI) | (int(r["ready"]) << 1) | (r["event"] << 2) | (int(r["hf"]) << 3)
        c |= (1 if r["sig"] == 1 else (2 if r["sig"] == -1 else 0)) << 4
        c |= int(r["thr"]) << 6
        c |= int(r["level"] == HI) << 7
        out.append(c)
    return np.array(out, dtype=np.uint8)


def replay_wallclock_prefix(D, w, k, inc, dec, C, hf_thr, *, dt=0.1, bw_max=20.0, f_min=0.8, f_max=2.2,
                            p_idle=60.0, p_core=40.0, p_umin=16.0, p_umax=100.0, p_gpu=87.0, kind="magus",
                            tdp=270.0, margin=0.05, c_dram=0.5, observe=0):
    """NEXT-1 wall-clock rounds (A32), re-stated independently: the work done inside a round is kept
    in exact rational arithmetic (fractions.Fraction) and each entry's duration is its exact dilation
    w + (1 - w) * D / A rounds; the governor samples the entry in progress at the start of each round and
    decides exactly as replay_prefix does, from the full prefix of observed samples and flags."""
    from fractions import Fraction as Fr
    B = {LO: f32(bw_max * (f_min / f_max)), HI: f32(bw_max * (f_max / f_max))}
    P = {LO: (p_idle + p_core) + p_umin, HI: (p_idle + p_core) + (p_umin + (p_umax - p_umin) * 1.0)}
    f = LO if kind in ("magus", "static_min") else HI
    D = [f32(d) for d in D]

    def dur(d, lev):                                         # rounds one whole entry takes at level lev
        a = d if observe else min(d, B[lev])
        if a < d:
            return Fr(f32(w)) + (1 - Fr(f32(w))) * Fr(d) / Fr(a)
        return Fr(1)

    observed, flags, rows, used_all = [], [], [], []
    e, left = 0, None                                        # entry in progress, its remaining duration (rounds)
    while e < len(D):
        d = D[e]
        a = d if observe else min(d, B[f])
        thr = a < d
        if left is None:
            left = dur(d, f)
        budget = Fr(1)
        while budget > 0 and e < len(D):
            if left > budget:
                left -= budget                               # (the remaining work keeps its fraction of the entry)
                budget = Fr(0)
            else:
                budget -= left
                e += 1
                left = dur(D[e], f) if e < len(D) else None
        used_all.append((f, 1 - budget))
        observed.append(a)
        sig, ready, hf = 0, False, False
        if kind == "magus":
            if len(observed) >= k + 1:
                ready = True
                deriv = (observed[-1] - observed[-1 - k]) / (k * dt)
                sig = 1 if deriv > inc else (-1 if deriv < dec else 0)
                flags.append(1 if sig != 0 else 0)
            if len(flags) >= C:
                window = flags[-C:]
                hf = (sum(window) / len(window)) >= hf_thr
            cmd = HI if hf else (HI if sig == 1 else (LO if sig == -1 else f))
        elif kind == "tdp":
            cmd = LO if (P[f] + c_dram * a) >= (1.0 - margin) * tdp else HI
        else:
            cmd = f
        rows.append(dict(level=f, cmd=cmd, ready=ready, event=int(ready and sig != 0), hf=hf, sig=sig, thr=thr))
        if cmd != f and left is not None:
            # the entry in progress continues at the new level: its remaining WORK fraction is kept
            frac = left / dur(D[e], f)
            left = frac * dur(D[e], cmd)
        f = cmd
    T = math.fsum(float(u) * dt for _, u in used_all)
    return rows, dict(T=T, E_pkg=math.fsum(P[l] * float(u) * dt for l, u in used_all),
                      E=math.fsum((P[l] + p_gpu) * float(u) * dt for l, u in used_all))
