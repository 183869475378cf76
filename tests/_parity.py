"""Helpers for the GPU-vs-oracle parity tests (test infrastructure).

The CUDA path is called through the C ABI (paper_2502_03796_b200.magus); the oracle through
oracle/oracle.py.  They share only the policy/model *parameters* built here from plain dicts.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O

EXACT = ["n_hi", "n_thr", "transitions", "tune_events", "lock_ticks", "digest"]
FLOAT = ["T", "E_pkg", "E", "EDP"]
FRACTIONS = ["slowdown", "energy_saving", "edp_saving", "pkg_power_saving"]
RTOL = 1e-9        # north_star: fp64 energy/EDP within 1e-9 relative
ATOL = 1e-12
# slowdown and the savings are 1 - ratio (or ratio - 1) of two such sums: 1e-9 relative on the ratio is
# 1e-9 absolute on the fraction; a relative bar would be meaningless at 0.
FRAC_ATOL = 1e-9


def gpu_policies(dicts):
    from paper_2502_03796_b200 import magus as M
    return [M.Policy(**d) for d in dicts]


def oracle_policies(dicts):
    return [O.Policy(**d) for d in dicts]


def gpu_model(**kw):
    from paper_2502_03796_b200 import magus as M
    return M.Model(**kw)


def oracle_model(**kw):
    return O.Model(**kw)


def compare_records(gpu_rec, ora_rec, label=""):
    """gpu_rec: structured [n][P] (magus_trace_stats); ora_rec: structured [n][P] (oracle OResult)."""
    assert gpu_rec.shape == ora_rec.shape, (gpu_rec.shape, ora_rec.shape)
    for k in EXACT:
        g, o = gpu_rec[k], ora_rec[k]
        bad = np.argwhere(g != o)
        assert bad.size == 0, f"{label} {k}: {len(bad)} mismatches, first (trace, policy) {bad[0].tolist()}: " \
                              f"gpu {g[tuple(bad[0])]} oracle {o[tuple(bad[0])]}"
    for k in FLOAT:
        g, o = gpu_rec[k], ora_rec[k]
        ok = np.isclose(g, o, rtol=RTOL, atol=ATOL)
        bad = np.argwhere(~ok)
        assert bad.size == 0, f"{label} {k}: {len(bad)} outside 1e-9, first {bad[0].tolist()}: " \
                              f"gpu {g[tuple(bad[0])]!r} oracle {o[tuple(bad[0])]!r}"
    for k in FRACTIONS:
        g, o = gpu_rec[k], ora_rec[k]
        bad = np.argwhere(np.abs(g - o) > FRAC_ATOL)
        assert bad.size == 0, f"{label} {k}: {len(bad)} differ by more than 1e-9, first {bad[0].tolist()}: " \
                              f"gpu {g[tuple(bad[0])]!r} oracle {o[tuple(bad[0])]!r}"


def pack_words(codes):
    """codes [n_samples][n][P] uint8 (oracle) -> words [P][n][n_blocks][2] uint32 (cmd, tune flag),
    tick 32b+i at bit 31-i, partial last block zero-padded."""
    n_samples, n, P = codes.shape
    nb = (n_samples + 31) // 32
    pad = nb * 32 - n_samples
    c = np.concatenate([codes, np.zeros((pad, n, P), np.uint8)], axis=0).reshape(nb, 32, n, P)
    weights = (1 << (31 - np.arange(32, dtype=np.uint64))).reshape(1, 32, 1, 1)
    cmd = ((c & 1).astype(np.uint64) * weights).sum(axis=1)
    ev = (((c >> 2) & 1).astype(np.uint64) * weights).sum(axis=1)
    out = np.stack([cmd, ev], axis=-1).astype(np.uint32)      # [nb][n][P][2]
    return np.transpose(out, (2, 1, 0, 3)).copy()             # [P][n][nb][2]


def pack_words_tpn(codes):
    """codes [n][P][n_samples] uint8 (oracle.gen_replay_codes layout) -> words [P][n][n_blocks][2] uint32
    (cmd, tune flag), tick 32b+i at bit 31-i, partial last block zero-padded."""
    n, P, ns = codes.shape
    nb = (ns + 31) // 32
    out = np.empty((P, n, nb, 2), np.uint32)
    for bit, slot in ((0, 0), (2, 1)):
        b = ((codes >> bit) & 1).astype(np.uint8)
        if nb * 32 != ns:
            b = np.concatenate([b, np.zeros((n, P, nb * 32 - ns), np.uint8)], axis=2)
        packed = np.packbits(b, axis=2, bitorder="big")              # [n][P][nb * 4] bytes, tick 0 at the MSB
        words = packed.reshape(n, P, nb, 4).view(">u4")[..., 0]        # big-endian: byte 0 holds ticks 0-7
        out[..., slot] = np.transpose(words, (1, 0, 2))
    return out


def compare_totals(gpu_totals, ora_rec, label=""):
    """Per-policy totals (MAGUS_TOT_*) against the oracle's (math.fsum of its records): E, E_pkg, T, EDP and the
    counts within 1e-9 relative; the three fraction columns (slowdown, energy_saving, edp_saving) are SUMS of
    n per-trace fractions, each held to 1e-9 absolute (FRAC_ATOL), so their bar is n * 1e-9 absolute."""
    want = oracle_totals(ora_rec)
    n = ora_rec.shape[0]
    frac = [4, 5, 6]
    other = [i for i in range(want.shape[1]) if i not in frac]
    np.testing.assert_allclose(gpu_totals[:, other], want[:, other], rtol=RTOL, atol=ATOL, err_msg=label)
    np.testing.assert_allclose(gpu_totals[:, frac], want[:, frac], rtol=0, atol=max(1, n) * FRAC_ATOL, err_msg=label)


def oracle_totals(ora_rec):
    """Per-policy sums the library reports (MAGUS_TOT_*), from oracle per-trace records (math.fsum)."""
    import math
    n, P = ora_rec.shape
    names = ["E", "E_pkg", "T", "EDP", "slowdown", "energy_saving", "edp_saving", "n_hi", "n_thr", "transitions",
             "tune_events", "lock_ticks"]
    out = np.zeros((P, 13))
    for p in range(P):
        for i, k in enumerate(names):
            out[p, i] = math.fsum(float(x) for x in ora_rec[k][:, p])
        out[p, 12] = n
    return out


def oracle_wallclock(tr_host, w_host, policies, n_traces, model, dump=(0, 0)):
    """NEXT-1 (A32): the oracle's wall-clock replay of every (trace, policy) chain -> (records [n][P] in the
    oracle's record dtype, codes [n_samples][dump n][P] of the first n_samples rounds of the dump window)."""
    from oracle import oracle as O
    ns = tr_host.shape[0]
    pols = oracle_policies(policies)
    rec = np.zeros((n_traces, len(pols)), dtype=O.RESULT_DTYPE)
    codes = np.zeros((ns, dump[1], len(pols)), np.uint8)
    for j in range(n_traces):
        col = np.ascontiguousarray(tr_host[:, j])
        for p, pp in enumerate(pols):
            want = dump[0] <= j < dump[0] + dump[1]
            r, c = O.replay_wallclock(col, float(w_host[j]), pp, model, codes=want)
            for f in O.RESULT_DTYPE.names:
                if not f.startswith("_"):
                    rec[j, p][f] = r[f]
            if want:
                codes[:, j - dump[0], p] = c[:ns]
    return rec, codes
