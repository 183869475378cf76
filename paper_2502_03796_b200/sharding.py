"""Host-side sharding of the replay over ranks.  No arithmetic of the method.

Weak scaling (bench): rank r owns global traces [r * n_per_rank, (r + 1) * n_per_rank).
Strong scaling (library users): a fixed total split into contiguous, near-equal ranges.
Traces are generated counter-based from their global id, so a shard's bytes equal the
single-process bytes; per-trace results are per global id; the only exchange is the per-policy
totals (one allreduce, sum), after which every rank computes the same argmin.
"""
from __future__ import annotations


def weak_shard(n_per_rank: int, rank: int, world: int):
    """(global_trace_offset, n_traces) of `rank` when every rank processes n_per_rank traces."""
    if not (0 <= rank < world) or n_per_rank < 0:
        raise ValueError("need 0 <= rank < world and n_per_rank >= 0")
    return rank * n_per_rank, n_per_rank


def strong_shard(n_total: int, rank: int, world: int):
    """(global_trace_offset, n_traces) of `rank` for a fixed total: contiguous ranges, sizes differ by <= 1."""
    if not (0 <= rank < world) or n_total < 0:
        raise ValueError("need 0 <= rank < world and n_total >= 0")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def argmin_edp(totals, edp_index: int = 3) -> int:
    """Argmin over policies of the total EDP, ties -> lowest index (A23)."""
    best, bv = 0, totals[0][edp_index]
    for p in range(1, len(totals)):
        if totals[p][edp_index] < bv:
            best, bv = p, totals[p][edp_index]
    return best
