"""World-size-2 host logic of the multi-GPU path on CPU (gloo), through the LIBRARY's host-only calls
(magus_grid_plan, magus_totals_argmin; include/magus_replay.h): the 2-D (trace x parameter-grid) plan,
shard-invariant inputs, the one exchange -- every rank's per-policy totals placed at its policy offset in the
global [P][13], summed by an allreduce -- and the argmin every rank then takes, against the single process
(DESIGN.md section 10).  The per-rank partials come from the oracle (test infrastructure: there is no GPU
here); on a GPU the library computes them and the allreduce is NCCL inside the run's graph.  -m "not gpu"."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_03796_b200 import magus as M
from paper_2502_03796_b200.sharding import weak_shard, strong_shard, grid_shard, argmin_edp
from paper_2502_03796_b200.configs import CONFIGS

NAMES = ["E", "E_pkg", "T", "EDP", "slowdown", "energy_saving", "edp_saving", "n_hi", "n_thr", "transitions",
         "tune_events", "lock_ticks"]


def test_shard_ranges():
    for n, world in ((4096, 8), (10, 3), (1, 4), (0, 2), (65536, 8)):
        shards = [strong_shard(n, r, world) for r in range(world)]
        assert sum(c for _, c in shards) == n
        assert all(shards[r][0] + shards[r][1] == shards[r + 1][0] for r in range(world - 1))
        assert max(c for _, c in shards) - min(c for _, c in shards) <= 1
    assert [weak_shard(4096, r, 8) for r in range(3)] == [(0, 4096), (4096, 4096), (8192, 4096)]
    with pytest.raises(ValueError):
        strong_shard(10, 3, 3)


@pytest.mark.parametrize("world,ps,n,P", [(8, 8, 1024, 65), (8, 2, 1024, 65), (8, 1, 65536, 2), (6, 3, 37, 7),
                                          (4, 4, 5, 4), (1, 1, 0, 1)])
def test_grid_plan_covers_every_trace_policy_pair_once(world, ps, n, P):
    """magus_grid_plan: over all ranks, every (trace, policy) pair is owned by exactly one rank; trace and
    policy ranges are contiguous with sizes differing by at most one; bad plans are refused."""
    owned = np.zeros((n, P), np.int32)
    for r in range(world):
        t0, nt, p0, npol = grid_shard(n, P, r, world, ps)
        owned[t0:t0 + nt, p0:p0 + npol] += 1
    assert np.all(owned == 1)
    cols = [grid_shard(n, P, r, world, ps)[3] for r in range(ps)]
    assert max(cols) - min(cols) <= 1
    for w, r, p in ((world, world, ps), (world, 0, P + 1), (world, 0, 0), (world + 1, 0, world)):
        if p < 1 or p > P or r >= w or w % p:
            with pytest.raises(ValueError):
                grid_shard(n, P, r, w, p)


def test_library_argmin_semantics():
    """magus_totals_argmin (A23): least total EDP, ties -> lowest index, policies without traces skipped
    (all considered when none has traces)."""
    t = np.zeros((5, M.N_TOTALS))
    t[:, 12] = 10
    t[:, 3] = [5.0, 3.0, 3.0, 4.0, 9.0]
    assert argmin_edp(t) == 1
    t[1, 12] = 0                    # policy 1 replayed no traces (another rank's slice, no exchange)
    assert argmin_edp(t) == 2
    t[:, 12] = 0
    t[:, 3] = 0
    assert argmin_edp(t) == 0


def _oracle_totals(offset, n, ns, policies, p_off, P_glob):
    """This rank's per-policy totals (oracle records of its traces x its policy slice), placed at its policy
    offset in the global [P_glob][13] (rows of other slices 0) -- what the library's chunk-sum kernel writes."""
    from oracle import oracle as O
    c = CONFIGS[5]
    desc = O.GenDesc(seed=c["seed"], n_traces=n, n_samples=ns, class_mix=c["class_mix"], global_trace_offset=offset)
    tr, w = O.gen_traces(desc)
    rec, _, _ = O.replay_batch(tr, w, [O.Policy(**d) for d in policies])
    tot = np.zeros((P_glob, 13))
    for p in range(len(policies)):
        tot[p_off + p] = [rec[k][:, p].astype(np.float64).sum() for k in NAMES] + [n]
    return tot, rec


POLS = CONFIGS[5]["policies"] + [dict(CONFIGS[5]["policies"][0], deriv_ticks=2, high_freq_threshold=0.4)]


def _worker(rank, world, port, n_total, ns, ps, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t0, nt, p0, npol = grid_shard(n_total, len(POLS), rank, world, ps)
    tot, rec = _oracle_totals(t0, nt, ns, POLS[p0:p0 + npol], p0, len(POLS))
    t = torch.tensor(tot, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    am = argmin_edp(t.numpy())                     # the library's argmin on every rank
    np.save(os.path.join(out_dir, f"tot{rank}.npy"), t.numpy())
    np.save(os.path.join(out_dir, f"dig{rank}.npy"), rec["digest"])
    np.save(os.path.join(out_dir, f"am{rank}.npy"), np.array([am]))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ps", [1, 2])
def test_two_rank_allreduce_equals_single_process(tmp_path, ps):
    """ps = 1: traces split 19 + 18 (ragged); ps = 2: the parameter grid split 3 + 2 policies, every rank all
    37 traces.  Totals after the allreduce and the library argmin equal the single process on both ranks."""
    n_total, ns = 37, 3000
    mp.spawn(_worker, args=(2, _free_port(), n_total, ns, ps, str(tmp_path)), nprocs=2, join=True)
    single, rec = _oracle_totals(0, n_total, ns, POLS, 0, len(POLS))
    for r in range(2):
        t = np.load(tmp_path / f"tot{r}.npy")
        np.testing.assert_allclose(t, single, rtol=1e-12)
        assert int(np.load(tmp_path / f"am{r}.npy")[0]) == argmin_edp(single)
    d0, d1 = np.load(tmp_path / "dig0.npy"), np.load(tmp_path / "dig1.npy")
    if ps == 1:   # per-trace results are per global id: the shards' digests concatenate to the single process
        assert np.array_equal(np.concatenate([d0, d1]), rec["digest"])
    else:         # policy slices: the ranks' digests are the single process's columns
        assert np.array_equal(np.concatenate([d0, d1], axis=1), rec["digest"])
