"""Full-size parity (VERDICT r1 "close the parity holes"): the bench's own
device-generated inputs against the oracle's host generator, the whole
config-B table against the oracle, a config-E shard (m = 10M / 8) against the
oracle, and a config-E-scale reference-sharded search (8 shards run one after
another on one GPU, merged on the device) bitwise equal to one search over all
10M references (SURVEY.md 8(e) "Determinism").

Reference anchors (paths relative to /root/reference/proj): bruteforce.cpp:42-100
(the search), rng.hpp:9-28 / bench.cpp:39-46,93-94 (input conventions),
bruteforce.cpp:81-96 (the reference axis that the shards split).
"""
import numpy as np
import pytest

from oracle.oracle import compare

pytestmark = pytest.mark.gpu


def _seeds(oracle, m, n, d):
    return oracle.derive_seed(42, m, d, 0), oracle.derive_seed(42, n, d, 1)


def _device_uniform(knn, torch, rows, d, seed, offset=0):
    x = torch.empty((rows, d), dtype=torch.float32, device="cuda")
    knn.fill_uniform_device(x.data_ptr(), rows * d, seed, offset)
    return x


@pytest.mark.parametrize("count,offset", [(1, 0), (1000003, 0), (4096, 123456789), (77, 1 << 40)])
def test_fill_uniform_device_matches_oracle_counter(knn, oracle, count, offset):
    """knn_b200_fill_uniform_device (bench.py's GPU inputs) == ko_fill_counter_f32
    (the reference arm's / oracle's inputs), bit for bit."""
    import torch
    seed = oracle.derive_seed(42, count, 1, 0)
    x = torch.empty(count, dtype=torch.float32, device="cuda")
    knn.fill_uniform_device(x.data_ptr(), count, seed, offset)
    torch.cuda.synchronize()
    host = oracle.counter_f32(1, count, seed, row_begin=0) if offset == 0 else None
    if host is None:
        out = np.empty(count, np.float32)
        oracle.lib.ko_fill_counter_f32(out, offset, count, seed)
        host = out
    got = x.cpu().numpy().reshape(-1)
    assert (got.view(np.uint32) == host.reshape(-1).view(np.uint32)).all()
    assert got.min() >= 0.0 and got.max() < 1.0


def test_config_b_full_table_vs_oracle(knn, oracle):
    """Config B (m = n = 38400, d = 96, k = 20), the bench's inputs and call
    (device-resident index, caller stream): all 38,400 queries against the
    oracle with the north-star comparator."""
    import torch
    m = n = 38400
    d, k = 96, 20
    sr, sq = _seeds(oracle, m, n, d)
    R = _device_uniform(knn, torch, m, d, sr)
    Q = _device_uniform(knn, torch, n, d, sq)
    s = torch.cuda.Stream()
    od = torch.empty((n, k), dtype=torch.float32, device="cuda")
    oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
    ix.search_device(Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(), stream=s.cuda_stream)
    s.synchronize()
    assert knn.last_fallback_count() == 0
    Rh = oracle.counter_f32(m, d, sr)
    Qh = oracle.counter_f32(n, d, sq)
    assert (R.cpu().numpy().view(np.uint32) == Rh.view(np.uint32)).all()
    ri, rd = oracle.knn(Qh, Rh, k)
    rep = compare(oi.cpu().numpy(), od.cpu().numpy(), ri, rd, Qh, Rh, oracle=oracle)
    assert rep.ok, rep
    ix.close()


def test_config_e_shard_vs_oracle(knn, oracle):
    """One config-E shard (m = 1.25M = 10M / 8, d = 128, k = 20) searched with
    8192 queries; 512 of them (spread over every query tile pair's range)
    checked against the oracle.  Rows are the global config-E rows of shard 3
    (counter stream offset), returned with global indices."""
    import torch
    M, d, k = 10_000_000, 128, 20
    shard = 3
    ms = M // 8
    lo = shard * ms
    n = 8192
    sr, sq = _seeds(oracle, M, 100_000, d)
    R = _device_uniform(knn, torch, ms, d, sr, offset=lo * d)
    Q = _device_uniform(knn, torch, n, d, sq)
    od = torch.empty((n, k), dtype=torch.float32, device="cuda")
    oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    ix = knn.Index(device_ptr=R.data_ptr(), m=ms, d=d, index_base=lo)
    ix.search_device(Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr())
    torch.cuda.synchronize()
    assert knn.last_fallback_count() == 0
    pick = np.linspace(0, n - 1, 512).astype(np.int64)
    Rh = R.cpu().numpy()
    Qh = Q.cpu().numpy()[pick]
    ri, rd = oracle.knn(Qh, Rh, k)
    rep = compare(oi.cpu().numpy()[pick] - lo, od.cpu().numpy()[pick], ri, rd, Qh, Rh,
                  oracle=oracle)
    assert rep.ok, rep
    ix.close()


def test_config_e_sharded_merge_is_bitwise_single_search(knn, oracle):
    """Config-E scale (m = 10M, n = 100K, d = 128, k = 20): the R-sharded
    search of a G = 8 run -- each shard searched with its global index base
    and raw keys, then knn_b200_merge_device -- equals one search over all 10M
    references bit for bit, and a query sample matches the oracle."""
    import torch
    M, n, d, k, G = 10_000_000, 100_000, 128, 20, 8
    sr, sq = _seeds(oracle, M, n, d)
    R = _device_uniform(knn, torch, M, d, sr)
    Q = _device_uniform(knn, torch, n, d, sq)
    full_d = torch.empty((n, k), dtype=torch.float32, device="cuda")
    full_i = torch.empty((n, k), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    ix = knn.Index(device_ptr=R.data_ptr(), m=M, d=d)
    ix.search_device(Q.data_ptr(), n, k, full_d.data_ptr(), full_i.data_ptr())
    torch.cuda.synchronize()
    ix.close()
    keys = torch.empty((G, n, k), dtype=torch.float32, device="cuda")
    idxs = torch.empty((G, n, k), dtype=torch.int64, device="cuda")
    from paper_0804_1448_b200.sharding import shard_bounds
    for g in range(G):
        lo, hi = shard_bounds(M, G, g)
        sx = knn.Index(device_ptr=R[lo:hi].data_ptr(), m=hi - lo, d=d, index_base=lo)
        sx.search_device(Q.data_ptr(), n, k, keys[g].data_ptr(), idxs[g].data_ptr(),
                         raw_keys=True)
        torch.cuda.synchronize()
        sx.close()
    md = torch.empty((n, k), dtype=torch.float32, device="cuda")
    mi = torch.empty((n, k), dtype=torch.int64, device="cuda")
    knn.merge_device(keys.data_ptr(), idxs.data_ptr(), G, n, k, md.data_ptr(), mi.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(mi, full_i)
    assert torch.equal(md.view(torch.int32), full_d.view(torch.int32))
    pick = np.linspace(0, n - 1, 48).astype(np.int64)
    Rh = R.cpu().numpy()
    Qh = Q.cpu().numpy()[pick]
    ri, rd = oracle.knn(Qh, Rh, k)
    rep = compare(mi.cpu().numpy()[pick], md.cpu().numpy()[pick], ri, rd, Qh, Rh, oracle=oracle)
    assert rep.ok, rep
