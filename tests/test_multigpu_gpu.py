"""The library's multi-GPU APIs on the one GPU this run has:
the single-process sharded handle (reference- and query-sharded) and the
one-process-per-GPU communicator path, both through NCCL (loaded by the
library).  With G = 1 the NCCL all-gather is the identity and the merge is a
1-way merge, so each must reproduce the plain search bit for bit; the G > 1
reference-sharded determinism is covered by test_scale_gpu (8 shards merged
on one device)."""
import numpy as np
import pytest

from oracle.oracle import compare

pytestmark = pytest.mark.gpu


def test_nccl_loads(knn):
    v = knn.nccl_version()
    assert v >= 22700, v


@pytest.mark.parametrize("mode", ["references", "queries"])
def test_sharded_handle_one_device(knn, oracle, mode):
    m, n, d, k = 20000, 1500, 48, 20
    R = oracle.uniform_f32(m, d, 71)
    Q = oracle.uniform_f32(n, d, 72)
    md = knn.SHARD_REFERENCES if mode == "references" else knn.SHARD_QUERIES
    h = knn.Sharded(R, 1, mode=md)
    t = h.search(Q, k)
    ref = knn.bf_knn(Q, R, k)
    assert (t.index == ref.index).all() and (t.distance == ref.distance).all()
    h.close()
    with pytest.raises(ValueError):
        knn.Sharded(R, 0)


def test_comm_dist_search_world_one(knn, oracle):
    """knn_b200_dist_search_device on a 1-rank communicator: local shard search
    (raw keys, global indices), ncclAllGather, device merge."""
    import torch
    m, n, d, k = 30000, 2000, 64, 16
    R = torch.from_numpy(oracle.uniform_f32(m, d, 81)).cuda()
    Q = torch.from_numpy(oracle.uniform_f32(n, d, 82)).cuda()
    uid = knn.nccl_unique_id()
    assert len(uid) == 128
    comm = knn.Comm(uid, 1, 0, 0)
    ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
    od = torch.empty((n, k), device="cuda")
    oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    comm.search_device(ix, Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(), stream=s.cuda_stream)
    s.synchronize()
    ref = knn.bf_knn(Q.cpu().numpy(), R.cpu().numpy(), k)
    assert (oi.cpu().numpy() == ref.index).all()
    assert (od.cpu().numpy() == ref.distance).all()
    comm.close()
    ix.close()
