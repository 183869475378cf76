"""World-size-2 host logic of the multi-GPU path on CPU (gloo): shard ranges, shard-invariant inputs,
and the one exchange -- the allreduce of per-policy totals, then the argmin on every rank -- equal the
single-process result.  The per-rank partials come from the oracle (test
infrastructure); the GPU path's own allreduce is NCCL inside the library.  -m "not gpu"."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_03796_b200.sharding import weak_shard, strong_shard, argmin_edp
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


def _partial_totals(offset, n, ns):
    from oracle import oracle as O
    c = CONFIGS[5]
    desc = O.GenDesc(seed=c["seed"], n_traces=n, n_samples=ns, class_mix=c["class_mix"], global_trace_offset=offset)
    tr, w = O.gen_traces(desc)
    rec, _, _ = O.replay_batch(tr, w, [O.Policy(**d) for d in c["policies"]])
    tot = np.array([[rec[k][:, p].astype(np.float64).sum() for k in NAMES] + [n] for p in range(len(c["policies"]))])
    return tot, rec


def _worker(rank, world, port, n_total, ns, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    offset, n = strong_shard(n_total, rank, world)
    tot, rec = _partial_totals(offset, n, ns)
    t = torch.tensor(tot, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    am = argmin_edp(t.numpy())
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


def test_two_rank_allreduce_equals_single_process(tmp_path):
    n_total, ns = 37, 3000      # ragged split 19 + 18
    mp.spawn(_worker, args=(2, _free_port(), n_total, ns, str(tmp_path)), nprocs=2, join=True)
    single, rec = _partial_totals(0, n_total, ns)
    for r in range(2):
        t = np.load(tmp_path / f"tot{r}.npy")
        np.testing.assert_allclose(t, single, rtol=1e-12)
        assert int(np.load(tmp_path / f"am{r}.npy")[0]) == argmin_edp(single)
    # per-trace results are per global id: the shards' digests concatenate to the single-process ones
    d = np.concatenate([np.load(tmp_path / "dig0.npy"), np.load(tmp_path / "dig1.npy")])
    assert np.array_equal(d, rec["digest"])
