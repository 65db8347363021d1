"""Multi-rank host logic on CPU with the gloo backend (world_size 2): the
sharding plan, global index bases, the all-gather layout and the merge
semantics of the reference-sharded search.  The per-rank device search and the
device merge kernel are replaced by the oracle here (they are covered by the
GPU tests); what is checked is that the distributed plumbing reproduces a
single search over all of R exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0804_1448_b200.sharding import check_shardable, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_topk(Q, R, lo, k):
    """Rank-local exact top-k: raw squared keys (double), global indices."""
    d2 = ((Q[:, None, :].astype(np.float64) - R[None, :, :].astype(np.float64)) ** 2).sum(-1)
    order = np.lexsort((np.arange(R.shape[0])[None, :].repeat(Q.shape[0], 0), d2), axis=1)[:, :k]
    keys = np.take_along_axis(d2, order, 1)
    return keys, order + lo


def _merge(keys, idx, k):
    """(key, index)-ordered k-way merge of rank lists (merge_kernel.cu semantics)."""
    n = keys.shape[1]
    K = keys.transpose(1, 0, 2).reshape(n, -1)
    I = idx.transpose(1, 0, 2).reshape(n, -1)
    order = np.lexsort((I, K), axis=1)[:, :k]
    return np.take_along_axis(K, order, 1), np.take_along_axis(I, order, 1)


def _worker(rank, world, port, Q, R, k, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = R.shape[0]
    check_shardable(m, world, k)
    lo, hi = shard_bounds(m, world, rank)
    keys, idx = _local_topk(Q, R[lo:hi], lo, k)
    kt = torch.from_numpy(keys)
    it = torch.from_numpy(idx)
    gk = [torch.empty_like(kt) for _ in range(world)]
    gi = [torch.empty_like(it) for _ in range(world)]
    dist.all_gather(gk, kt)
    dist.all_gather(gi, it)
    if rank == 0:
        mk, mi = _merge(torch.stack(gk).numpy(), torch.stack(gi).numpy(), k)
        out["keys"] = mk
        out["idx"] = mi
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_plan_matches_single_search(world):
    rng = np.random.default_rng(3)
    Q = rng.random((40, 7)).astype(np.float32)
    R = rng.random((301, 7)).astype(np.float32)
    R[150] = R[10]  # a cross-shard duplicate: the tie rule must pick index 10
    k = 9
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), Q, R, k, out), nprocs=world, join=True)
    ref_keys, ref_idx = _local_topk(Q, R, 0, k)
    assert (out["idx"] == ref_idx).all()
    assert (out["keys"] == ref_keys).all()


def test_shard_bounds_cover_and_balance():
    for m in (1, 7, 38400, 10_000_000):
        for world in (1, 2, 4, 8):
            b = [shard_bounds(m, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == m
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        check_shardable(10, 4, 3)
