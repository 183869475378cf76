"""Host-side sharding of the replay over ranks: thin wrappers of the library's
host-only magus_grid_plan / magus_totals_argmin (include/magus_replay.h).  No arithmetic of the method.

Weak scaling (bench): each trace shard holds n_per_rank traces, so the global trace count grows with the world.
Strong scaling: a fixed total cut into contiguous ranges whose sizes differ by at most one.
Parameter-grid split: policy_shards columns of the world each replay a contiguous slice of the policy set.
Traces are generated counter-based from their global id, so a shard's bytes equal the single-process bytes;
per-trace results are per global id; the only exchange is the per-policy totals (one allreduce over the
global [n_policies][13], sum), after which every rank takes the same argmin.
"""
from __future__ import annotations

from . import magus as M


def grid_shard(n_traces: int, n_policies: int, rank: int, world: int, policy_shards: int = 1):
    """(global_trace_offset, n_traces, policy_offset, n_policies) of `rank` (magus_grid_plan)."""
    try:
        return M.grid_plan(world, rank, policy_shards, n_traces, n_policies)
    except M.MagusError as e:
        raise ValueError(str(e)) from None


def weak_shard(n_per_rank: int, rank: int, world: int):
    """(global_trace_offset, n_traces) of `rank` when every rank processes n_per_rank traces."""
    if n_per_rank < 0:
        raise ValueError("n_per_rank must be >= 0")
    off, n, _, _ = grid_shard(n_per_rank * world, 1, rank, world)
    return off, n


def strong_shard(n_total: int, rank: int, world: int):
    """(global_trace_offset, n_traces) of `rank` for a fixed total: contiguous ranges, sizes differ by <= 1."""
    off, n, _, _ = grid_shard(n_total, 1, rank, world)
    return off, n


def argmin_edp(totals) -> int:
    """The library's argmin over policies of the total EDP (A23)."""
    return M.totals_argmin(totals)
