"""GPU parity tests: the CUDA engine (through the C ABI) against the oracle and
the reference's golden outputs, with the north-star tolerance comparator
(distances within 1e-5 relative; index differences only at near-ties).

Mirrors the reference's own hot-path tests (paths relative to
/root/reference/proj/tests): test_bruteforce.cpp (hand-checked KATs, contract
errors, random instances vs the serial oracle, determinism, evaluation count)
and acceptance.cpp C1 / C3 / C9.
"""
import numpy as np
import pytest

from oracle.oracle import CHEBYSHEV, EUCLIDEAN, MAHALANOBIS, MANHATTAN, compare

pytestmark = pytest.mark.gpu

PATHS = ("exact", "tensor", "auto")


def cfg(knn, path):
    p = {"exact": knn.PATH_EXACT, "tensor": knn.PATH_TENSOR, "auto": knn.PATH_AUTO}[path]
    return knn.BfConfig(path=p, device=0)


def metric_of(knn, kind, mahal=None):
    if kind == MAHALANOBIS:
        d = int(round(len(mahal) ** 0.5))
        return knn.Metric.mahalanobis(d, mahal)
    return knn.Metric(kind)


def check_invariants(table, m):
    """test_bruteforce.cpp:22-39: range, distinct, ascending, ties by index."""
    idx, dist = table.index, table.distance
    assert (idx >= 0).all() and (idx < m).all()
    for i in range(idx.shape[0]):
        assert len(set(idx[i].tolist())) == idx.shape[1]
        dd = dist[i]
        assert (np.diff(dd) >= 0).all()
        same = np.nonzero(np.diff(dd) == 0)[0]
        assert (idx[i][same + 1] > idx[i][same]).all()


@pytest.mark.parametrize("path", PATHS)
def test_golden_reference_outputs(knn, golden, oracle, path):
    """Every golden case (reference's own outputs, tests/golden/) within tolerance."""
    for name, c in golden.items():
        kind = int(c["metric"])
        mahal = c["mahal"] if kind == MAHALANOBIS else None
        t = knn.bf_knn(c["Q"], c["R"], int(c["k"]), metric_of(knn, kind, mahal),
                       config=cfg(knn, path))
        rep = compare(t.index, t.distance, c["idx"], c["dist"], c["Q"], c["R"], kind,
                      oracle=oracle, mahal=mahal, atol=1e-6)
        assert rep.ok, f"{name}: {rep}"
        check_invariants(t, c["R"].shape[0])


@pytest.mark.parametrize("path", PATHS)
def test_collinear_and_full_sort(knn, path):
    # test_bruteforce.cpp:77-90
    R = np.array([[0, 0], [1, 0], [2, 0]], np.float32)
    Q = np.array([[0.1, 0]], np.float32)
    t = knn.bf_knn(Q, R, 2, config=cfg(knn, path))
    assert t.index[0].tolist() == [0, 1]
    assert t.distance[0, 0] == pytest.approx(0.1, rel=1e-6)
    assert t.distance[0, 1] == pytest.approx(0.9, rel=1e-6)
    full = knn.bf_knn(Q, R, 3, config=cfg(knn, path))
    assert full.index[0, 2] == 2
    check_invariants(full, 3)


@pytest.mark.parametrize("path", PATHS)
def test_all_duplicates_resolve_to_lowest_indices(knn, path):
    # test_kdtree.cpp:65-75
    P = np.full((64, 3), 1.5, np.float32)
    t = knn.bf_knn(np.full((1, 3), 1.5, np.float32), P, 5, config=cfg(knn, path))
    assert t.index[0].tolist() == [0, 1, 2, 3, 4]
    assert (t.distance == 0).all()


@pytest.mark.parametrize("path", PATHS)
def test_self_join_has_exact_zero_self_match(knn, oracle, path):
    # entropy.cpp:48-57 relies on the self match appearing at distance 0 in k+1
    P = oracle.uniform_f32(700, 24, 77)
    t = knn.bf_knn(P, P, 5, config=cfg(knn, path))
    assert (t.distance[:, 0] == 0).all()
    assert (t.index[:, 0] == np.arange(700)).all()


@pytest.mark.parametrize("metric", [EUCLIDEAN, MANHATTAN, CHEBYSHEV, MAHALANOBIS])
def test_random_instances_vs_oracle(knn, oracle, metric):
    """acceptance.cpp:58-84 style (C1), tolerance instead of bitwise."""
    rng = np.random.default_rng(1001 + metric)
    spd = np.array([2.0, 0.4, 0.0, 0.4, 1.5, -0.2, 0.0, -0.2, 1.0])
    for trial in range(25):
        n, m = int(rng.integers(1, 300)), int(rng.integers(1, 700))
        d = 3 if metric == MAHALANOBIS else int(rng.integers(1, 70))
        k = int(rng.integers(1, min(m, 300) + 1))
        Q = (rng.random((n, d)) * 10 - 5).astype(np.float32)
        R = (rng.random((m, d)) * 10 - 5).astype(np.float32)
        mahal = spd if metric == MAHALANOBIS else None
        ri, rd = oracle.knn(Q, R, k, metric, mahal)
        for path in PATHS:
            t = knn.bf_knn(Q, R, k, metric_of(knn, metric, mahal), config=cfg(knn, path))
            rep = compare(t.index, t.distance, ri, rd, Q, R, metric, oracle=oracle, mahal=mahal,
                          atol=1e-6)
            assert rep.ok, f"trial {trial} n={n} m={m} d={d} k={k} path={path}: {rep}"


@pytest.mark.parametrize("k", [1, 20, 100, 256, 1024])
def test_k_sweep_subsample(knn, oracle, k):
    """Config D shape (m=38400, d=64) on a 192-query subsample, k up to 1024."""
    m, d = 38400, 64
    R = oracle.uniform_f32(m, d, oracle.derive_seed(42, m, d, 0))
    Q = oracle.uniform_f32(192, d, oracle.derive_seed(42, m, d, 1))
    ri, rd = oracle.knn(Q, R, k)
    for path in PATHS:
        t = knn.bf_knn(Q, R, k, config=cfg(knn, path))
        rep = compare(t.index, t.distance, ri, rd, Q, R, oracle=oracle)
        assert rep.ok, f"k={k} path={path}: {rep}"


@pytest.mark.parametrize("d", [8, 16, 32, 64, 80, 96, 128])
def test_d_sweep_subsample(knn, oracle, d):
    """Config C shape (m=19200, k=20) on a 256-query subsample."""
    m = 19200
    R = oracle.uniform_f32(m, d, oracle.derive_seed(42, m, d, 0))
    Q = oracle.uniform_f32(256, d, oracle.derive_seed(42, m, d, 1))
    ri, rd = oracle.knn(Q, R, 20)
    for path in PATHS:
        t = knn.bf_knn(Q, R, 20, config=cfg(knn, path))
        rep = compare(t.index, t.distance, ri, rd, Q, R, oracle=oracle)
        assert rep.ok, f"d={d} path={path}: {rep}"


def test_config_a_full(knn, oracle):
    """BASELINE configs[0]: m=n=4800, d=32, k=20, every query."""
    R = oracle.uniform_f32(4800, 32, oracle.derive_seed(42, 4800, 32, 0))
    Q = oracle.uniform_f32(4800, 32, oracle.derive_seed(42, 4800, 32, 1))
    ri, rd = oracle.knn(Q, R, 20)
    for path in PATHS:
        t = knn.bf_knn(Q, R, 20, config=cfg(knn, path))
        rep = compare(t.index, t.distance, ri, rd, Q, R, oracle=oracle)
        assert rep.ok, f"path={path}: {rep}"


def test_config_b_subsample(knn, oracle):
    """BASELINE configs[1] (headline): m=n=38400, d=96, k=20; full search on the
    GPU, 512 queries checked against the oracle, the rest via invariants."""
    m = n = 38400
    d = 96
    R = oracle.uniform_f32(m, d, oracle.derive_seed(42, m, d, 0))
    Q = oracle.uniform_f32(n, d, oracle.derive_seed(42, n, d, 1))
    t = knn.bf_knn(Q, R, 20, config=cfg(knn, "auto"))
    sel = np.linspace(0, n - 1, 512).astype(int)
    ri, rd = oracle.knn(Q[sel], R, 20)
    rep = compare(t.index[sel], t.distance[sel], ri, rd, Q[sel], R, oracle=oracle)
    assert rep.ok, str(rep)
    check_invariants(t, m)


@pytest.mark.parametrize("k", [17, 150])
def test_paths_are_bitwise_identical(knn, oracle, k):
    """C3 analogue: exact / tensor / auto give bitwise-equal tables (k=17: the
    running-bound tensor path; k=150: the large-k fixed-threshold path)."""
    R = oracle.uniform_f32(9000, 40, 11)
    Q = oracle.uniform_f32(1000, 40, 12)
    tabs = [knn.bf_knn(Q, R, k, config=cfg(knn, p)) for p in PATHS]
    for t in tabs[1:]:
        assert (t.index == tabs[0].index).all()
        assert (t.distance == tabs[0].distance).all()


@pytest.mark.parametrize("metric", [EUCLIDEAN, MANHATTAN, CHEBYSHEV])
def test_exact_kernel_work_split_and_list_variants(knn, oracle, metric):
    """The exact SIMT kernel's stream-K split (a query block spread over many
    CTAs, one output slot per CTA, padded slots) and its list variants
    (register lists of 1/2/4 x 32 entries, global lists above 128), on ragged
    d (zero-filled coordinate tails) and partial last tiles."""
    cases = [(100, 20011, 33, 32), (100, 20011, 33, 33), (7, 9000, 1, 64), (129, 5000, 97, 65),
             (300, 3000, 31, 128), (60, 4100, 12, 129), (257, 700, 5, 1)]
    for (n, m, d, k) in cases:
        Q = oracle.uniform_f32(n, d, 300 + n) * 4 - 2
        R = oracle.uniform_f32(m, d, 400 + m) * 4 - 2
        ri, rd = oracle.knn(Q, R, k, metric)
        t = knn.bf_knn(Q, R, k, knn.Metric(metric), config=cfg(knn, "exact"))
        rep = compare(t.index, t.distance, ri, rd, Q, R, metric, oracle=oracle)
        assert rep.ok, f"{(n, m, d, k)} metric={metric}: {rep}"
        check_invariants(t, m)


def test_mahalanobis_device_whitening(knn, oracle):
    """Metric::whiten (metric.cpp:63-82) runs on the device for both the host
    and the device-resident API; both equal the oracle within tolerance and
    each other bitwise."""
    import torch
    rng = np.random.default_rng(77)
    d = 24
    A = rng.standard_normal((d, d))
    M = A @ A.T + d * np.eye(d)
    Q = (rng.random((300, d)) * 4 - 2).astype(np.float32)
    R = (rng.random((5000, d)) * 4 - 2).astype(np.float32)
    k = 15
    ri, rd = oracle.knn(Q, R, k, MAHALANOBIS, M.ravel())
    th = knn.bf_knn(Q, R, k, knn.Metric.mahalanobis(d, M.ravel()))
    rep = compare(th.index, th.distance, ri, rd, Q, R, MAHALANOBIS, oracle=oracle,
                  mahal=M.ravel(), atol=1e-6)
    assert rep.ok, str(rep)
    Qd = torch.from_numpy(Q).cuda()
    Rd = torch.from_numpy(R).cuda()
    od = torch.empty((300, k), device="cuda")
    oi = torch.empty((300, k), dtype=torch.int64, device="cuda")
    knn.search_device(Qd.data_ptr(), 300, Rd.data_ptr(), 5000, d, k, od.data_ptr(), oi.data_ptr(),
                      metric=MAHALANOBIS, mahalanobis=M)
    torch.cuda.synchronize()
    assert (oi.cpu().numpy() == th.index).all()
    assert (od.cpu().numpy() == th.distance).all()
    assert (Qd.cpu().numpy() == Q).all()  # caller's inputs untouched


def test_chunk_and_workers_do_not_change_results(knn, oracle):
    # test_bruteforce.cpp:124-136
    R = oracle.uniform_f32(53, 6, 102)
    Q = oracle.uniform_f32(37, 6, 101)
    base = knn.bf_knn(Q, R, 7)
    for workers in (1, 2, 8):
        for chunk in (1, 7, 37):
            t = knn.bf_knn(Q, R, 7, config=knn.BfConfig(chunk_size=chunk, worker_count=workers))
            assert (t.index == base.index).all() and (t.distance == base.distance).all()


def test_distance_evals_is_n_times_m(knn, oracle):
    # test_bruteforce.cpp:138-148 / acceptance C9
    R = oracle.uniform_f32(40, 4, 56)
    Q = oracle.uniform_f32(30, 4, 55)
    for k in (1, 20, 40):
        st = knn.SearchStats()
        knn.bf_knn(Q, R, k, config=knn.BfConfig(count_distance_evals=True), stats=st)
        assert st.distance_evals == 30 * 40
    st = knn.SearchStats(distance_evals=123)
    knn.bf_knn(Q, R, 3, stats=st)
    assert st.distance_evals == 0  # bruteforce.cpp:98 writes 0 when not counting


def test_sharded_merge_equals_single_search(knn, oracle):
    """R split into shards with global index bases, merged on device ==
    one search over all of R, bitwise (SURVEY.md 8(e) determinism)."""
    import torch
    m, d, n, k = 30000, 48, 800, 20
    R = oracle.uniform_f32(m, d, 5)
    Q = oracle.uniform_f32(n, d, 6)
    full = knn.bf_knn(Q, R, k)
    dev = torch.device("cuda:0")
    Qd = torch.from_numpy(Q).to(dev)
    bounds = [0, 7000, 19000, 30000]
    keys = torch.empty((3, n, k), dtype=torch.float32, device=dev)
    idxs = torch.empty((3, n, k), dtype=torch.int64, device=dev)
    for s in range(3):
        Rs = torch.from_numpy(R[bounds[s]:bounds[s + 1]].copy()).to(dev)
        ix = knn.Index(device_ptr=Rs.data_ptr(), m=Rs.shape[0], d=d, index_base=bounds[s])
        ix.search_device(Qd.data_ptr(), n, k, keys[s].data_ptr(), idxs[s].data_ptr(),
                         raw_keys=True)
        torch.cuda.synchronize()
        ix.close()
    od = torch.empty((n, k), dtype=torch.float32, device=dev)
    oi = torch.empty((n, k), dtype=torch.int64, device=dev)
    knn.merge_device(keys.data_ptr(), idxs.data_ptr(), 3, n, k, od.data_ptr(), oi.data_ptr())
    torch.cuda.synchronize()
    assert (oi.cpu().numpy() == full.index).all()
    assert (od.cpu().numpy() == full.distance).all()


def test_index_handle_host_roundtrip(knn, oracle):
    R = oracle.uniform_f32(5000, 20, 21)
    Q = oracle.uniform_f32(333, 20, 22)
    ix = knn.Index(R)
    a = ix.search(Q, 9)
    b = knn.bf_knn(Q, R, 9)
    assert (a.index == b.index).all() and (a.distance == b.distance).all()
    ix.close()


def test_large_d_and_odd_shapes(knn, oracle):
    for (n, m, d, k) in [(1, 1, 1, 1), (65, 129, 300, 129), (3, 5000, 513, 7), (130, 64, 2, 64)]:
        Q = oracle.uniform_f32(n, d, 1000 + d) * 3 - 1
        R = oracle.uniform_f32(m, d, 2000 + d) * 3 - 1
        ri, rd = oracle.knn(Q, R, k)
        for path in PATHS:
            t = knn.bf_knn(Q, R, k, config=cfg(knn, path))
            rep = compare(t.index, t.distance, ri, rd, Q, R, oracle=oracle)
            assert rep.ok, f"{(n, m, d, k)} {path}: {rep}"


def test_tensor_path_is_used_and_certified(knn, oracle):
    """Random data: every query certified by the tcgen05 candidate bound (no
    exact-kernel fallback).  Duplicate-heavy data: the candidate-group log
    holds every reference inside the bound, still certified and exact.  All
    references identical: every group passes the bound, a log overflows, the
    certificate fails and the exact kernel recomputes -- results still exact."""
    R = oracle.uniform_f32(20000, 96, 31)
    Q = oracle.uniform_f32(3000, 96, 32)
    t = knn.bf_knn(Q, R, 20, config=knn.BfConfig(path=knn.PATH_TENSOR))
    assert knn.last_fallback_count() == 0
    ri, rd = oracle.knn(Q[:300], R, 20)
    assert compare(t.index[:300], t.distance[:300], ri, rd, Q[:300], R, oracle=oracle).ok
    # 40 copies of every point: many exact ties inside the bound
    base = oracle.uniform_f32(100, 16, 33)
    Rd = np.repeat(base, 40, axis=0)
    Qd = oracle.uniform_f32(50, 16, 34)
    td = knn.bf_knn(Qd, Rd, 20, config=knn.BfConfig(path=knn.PATH_TENSOR))
    te = knn.bf_knn(Qd, Rd, 20, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (td.index == te.index).all() and (td.distance == te.distance).all()
    ri, rd = oracle.knn(Qd, Rd, 20)
    assert compare(td.index, td.distance, ri, rd, Qd, Rd, oracle=oracle).ok
    # one point repeated: every 8-reference group is a candidate -> log overflow
    Rs = np.repeat(oracle.uniform_f32(1, 16, 35), 80000, axis=0)
    ts = knn.bf_knn(Qd, Rs, 20, config=knn.BfConfig(path=knn.PATH_TENSOR))
    assert knn.last_fallback_count() > 0
    tse = knn.bf_knn(Qd, Rs, 20, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (ts.index == tse.index).all() and (ts.distance == tse.distance).all()
    assert (ts.index == np.arange(20)[None, :]).all()


@pytest.mark.gpu
def test_device_fallback_is_asynchronous_on_a_stream(knn, oracle):
    """Index search on a caller stream: the certification fallback (exact
    kernel over a device-side query list) runs without a host round trip, so
    the call returns before the work is done; after a stream sync the table is
    the exact one.  Mixed batch: uniform queries certify, queries sitting on a
    heavily duplicated reference overflow their logs and fall back."""
    import torch
    d, k = 16, 20
    base = oracle.uniform_f32(2000, d, 41)
    dup = np.repeat(oracle.uniform_f32(1, d, 42), 30000, axis=0)
    R = np.concatenate([base, dup]).astype(np.float32)
    Q = np.concatenate([oracle.uniform_f32(300, d, 43), dup[:40] + 1e-4]).astype(np.float32)
    n, m = Q.shape[0], R.shape[0]
    Qd, Rd = torch.from_numpy(Q).cuda(), torch.from_numpy(R).cuda()
    od = torch.empty((n, k), device="cuda")
    oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
    ix = knn.Index(device_ptr=Rd.data_ptr(), m=m, d=d)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ix.search_device(Qd.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(),
                         stream=s.cuda_stream)
    s.synchronize()
    assert knn.last_fallback_count() > 0
    te = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (oi.cpu().numpy() == te.index).all()
    assert (od.cpu().numpy() == te.distance).all()
    ix.close()


@pytest.mark.gpu
@pytest.mark.parametrize("k", [33, 64, 129, 500, 1000])
def test_large_k_block_sizes(knn, oracle, k):
    """The large-k selection picks 64 / 128 / 256-thread blocks from the
    candidate capacity; every size must give the exact table."""
    m, d = 12000, 24
    R = oracle.uniform_f32(m, d, 600 + k)
    Q = oracle.uniform_f32(128, d, 700 + k)
    ri, rd = oracle.knn(Q, R, k)
    t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    rep = compare(t.index, t.distance, ri, rd, Q, R, oracle=oracle)
    assert rep.ok, f"k={k}: {rep}"
    te = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (t.index == te.index).all() and (t.distance == te.distance).all()


@pytest.mark.gpu
def test_every_k_tensor_equals_exact(knn, oracle):
    """Every k from 1 to 40 (each bound-list size, the small/large switch)
    and large k up to 1024 on one shape: the tensor path's table is bitwise
    the exact path's on a query sample, with every query certified."""
    m, n, d = 20000, 2048, 29
    R = oracle.uniform_f32(m, d, 861)
    Q = oracle.uniform_f32(n, d, 862)
    rows = np.arange(0, n, 32)
    for k in list(range(1, 41)) + [64, 100, 129, 256, 500, 1024]:
        t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
        assert knn.last_fallback_count() == 0, f"k={k}"
        te = knn.bf_knn(Q[rows], R, k, config=knn.BfConfig(path=knn.PATH_EXACT))
        assert (t.index[rows] == te.index).all() and (t.distance[rows] == te.distance).all(), f"k={k}"


@pytest.mark.gpu
@pytest.mark.parametrize("k", [21, 28, 32])
def test_small_k_32_entry_lists(knn, oracle, k):
    """k = 21 .. 32 runs the filter with 32-entry bound lists (no batched
    drains), with several units per CTA: exact table, every query certified."""
    m, n, d = 20000, 2048, 29
    R = oracle.uniform_f32(m, d, 840 + k)
    Q = oracle.uniform_f32(n, d, 850 + k)
    t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    assert knn.last_fallback_count() == 0
    rows = np.arange(0, n, 16)
    ri, rd = oracle.knn(Q[rows], R, k)
    rep = compare(t.index[rows], t.distance[rows], ri, rd, Q[rows], R, oracle=oracle)
    assert rep.ok, f"k={k}: {rep}"
    te = knn.bf_knn(Q[rows], R, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (t.index[rows] == te.index).all() and (t.distance[rows] == te.distance).all()


@pytest.mark.gpu
@pytest.mark.parametrize("k", [100, 300])
def test_large_k_duplicate_ties(knn, oracle, k):
    """Large k on duplicate-heavy references (40 copies of each point): runs of
    40 equal exact keys overfill the select's buckets (<= 32 entries), so the
    bitonic sort of all candidates takes over; ties resolve by ascending index,
    bitwise the exact path's table."""
    base = oracle.uniform_f32(150, 16, 36)
    Rd = np.repeat(base, 40, axis=0)
    Qd = oracle.uniform_f32(64, 16, 37)
    td = knn.bf_knn(Qd, Rd, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    te = knn.bf_knn(Qd, Rd, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (td.index == te.index).all() and (td.distance == te.distance).all()
    ri, rd = oracle.knn(Qd, Rd, k)
    assert compare(td.index, td.distance, ri, rd, Qd, Rd, oracle=oracle).ok


@pytest.mark.gpu
@pytest.mark.parametrize("d", [8, 16, 32, 64, 128])
@pytest.mark.parametrize("k", [100, 256])
def test_large_k_certifies_uniform_data(knn, oracle, d, k):
    """On uniform data every query certifies at every d: the select's bound
    bins must cover negative A (= D^2 - |q~|^2, the low-d case) and its
    candidate capacity must hold the values inside thresh(B) -- a failure here
    is silent in the results (the exact fallback answers) but costs the exact
    path's time."""
    m, n = 20000, 256
    R = oracle.uniform_f32(m, d, 810 + d + k)
    Q = oracle.uniform_f32(n, d, 820 + d + k)
    t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    assert knn.last_fallback_count() == 0, f"d={d} k={k}: {knn.last_fallback_count()} fallbacks"
    rows = np.arange(0, n, 8)
    ri, rd = oracle.knn(Q[rows], R, k)
    rep = compare(t.index[rows], t.distance[rows], ri, rd, Q[rows], R, oracle=oracle)
    assert rep.ok, f"d={d} k={k}: {rep}"


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["huge", "tiny", "offset", "query_outside_range"])
def test_tensor_path_extreme_magnitudes(knn, oracle, case):
    """The fp16 filter's centre/scale and rounding radii under extreme
    coordinate magnitudes: results stay exact (certified, or recomputed by the
    exact kernel when a query overflows fp16 or the bound is too loose)."""
    rng = np.random.default_rng({"huge": 1, "tiny": 2, "offset": 3, "query_outside_range": 4}[case])
    m, n, d, k = 6000, 300, 24, 10
    R = rng.standard_normal((m, d))
    Q = rng.standard_normal((n, d))
    if case == "huge":
        R, Q = R * 1e18, Q * 1e18
    elif case == "tiny":
        R, Q = R * 1e-18, Q * 1e-18
    elif case == "offset":
        R, Q = R + 1e4, Q + 1e4
    else:
        Q = Q * 1e9
    R = R.astype(np.float32)
    Q = Q.astype(np.float32)
    ri, rd = oracle.knn(Q, R, k)
    t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    rep = compare(t.index, t.distance, ri, rd, Q, R, oracle=oracle)
    assert rep.ok, f"{case}: {rep}"


@pytest.mark.gpu
@pytest.mark.parametrize("k", [64, 300])
def test_large_k_fallback_on_device(knn, oracle, k):
    """Large k (fixed-threshold filter + block selection): one point repeated
    fills every log, the certificate fails for every query and the exact
    kernel recomputes them from the device-side query list (no host round
    trip) -- the table is the exact path's, bitwise."""
    Qd = oracle.uniform_f32(50, 16, 734)
    Rs = np.repeat(oracle.uniform_f32(1, 16, 735), 40000, axis=0)
    ts = knn.bf_knn(Qd, Rs, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    assert knn.last_fallback_count() > 0
    tse = knn.bf_knn(Qd, Rs, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (ts.index == tse.index).all() and (ts.distance == tse.distance).all()
    assert (ts.index == np.arange(k)[None, :]).all()


@pytest.mark.gpu
@pytest.mark.parametrize("k", [16, 100])
def test_index_search_captures_into_a_cuda_graph(knn, oracle, k):
    """An index search on a caller stream (no host round trip for any k,
    certification fallbacks included) can be captured into a CUDA graph;
    replays give the eager result bitwise."""
    import torch
    n, m, d = 2000, 20000, 40
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        Q = torch.from_numpy(oracle.uniform_f32(n, d, 91)).cuda()
        R = torch.from_numpy(oracle.uniform_f32(m, d, 92)).cuda()
        od = torch.empty((n, k), device="cuda")
        oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
        ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
        go = lambda: ix.search_device(Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(),
                                      stream=s.cuda_stream)
        go()
        s.synchronize()
        ref_i, ref_d = oi.clone(), od.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            go()
        od.zero_()
        oi.zero_()
        g.replay()
        s.synchronize()
    assert (oi == ref_i).all() and (od == ref_d).all()
    ri, rd = oracle.knn(Q.cpu().numpy()[:200], R.cpu().numpy(), k)
    assert compare(oi.cpu().numpy()[:200], od.cpu().numpy()[:200], ri, rd,
                   Q.cpu().numpy()[:200], R.cpu().numpy(), oracle=oracle).ok
    ix.close()


@pytest.mark.gpu
@pytest.mark.parametrize("metric", [EUCLIDEAN, MANHATTAN])
def test_full_sort_k_equals_m(knn, oracle, metric):
    """k = m (the full sort, test_bruteforce.cpp:86-89 at scale): global lists,
    merge scratch for k > 2048 and the exact path for k > 1024."""
    m, n, d = 2600, 20, 7
    R = oracle.uniform_f32(m, d, 801)
    Q = oracle.uniform_f32(n, d, 802)
    ri, rd = oracle.knn(Q, R, m, metric)
    t = knn.bf_knn(Q, R, m, knn.Metric(metric))
    rep = compare(t.index, t.distance, ri, rd, Q, R, metric, oracle=oracle)
    assert rep.ok, str(rep)
    check_invariants(t, m)


@pytest.mark.gpu
def test_non_finite_detected_on_device(knn, oracle):
    """The host API validates coordinates on the device copy (point_set.hpp:27-31
    text, first offending coordinate in row-major order)."""
    R = oracle.uniform_f32(3000, 32, 41)
    Q = oracle.uniform_f32(500, 32, 42)
    Qb = Q.copy()
    Qb[7, 3] = np.inf
    Qb[9, 1] = np.nan
    with pytest.raises(ValueError, match=r"^PointSet: non-finite coordinate at point 7, dimension 3$"):
        knn.bf_knn(Qb, R, 5)
    Rb = R.copy()
    Rb[2999, 31] = -np.inf
    with pytest.raises(ValueError, match=r"^PointSet: non-finite coordinate at point 2999, dimension 31$"):
        knn.bf_knn(Q, Rb, 5)
    # a clean search on the same context still works afterwards
    t = knn.bf_knn(Q, R, 5)
    ri, rd = oracle.knn(Q[:50], R, 5)
    assert compare(t.index[:50], t.distance[:50], ri, rd, Q[:50], R, oracle=oracle).ok


@pytest.mark.gpu
def test_non_finite_detected_device_api(knn, oracle):
    """The synchronous device-pointer API checks the caller's values first
    (PointSet semantics) with the 16-byte-load scan: the first offending
    coordinate is reported in the aligned middle, in the scalar head of a
    misaligned pointer and in the scalar tail."""
    import torch
    n, m, d, k = 300, 2000, 13, 5  # n*d, m*d not multiples of 4: scalar tails
    R = torch.from_numpy(oracle.uniform_f32(m, d, 43)).cuda()
    flat = torch.from_numpy(oracle.uniform_f32(n * d + 1, 1, 44).ravel()).cuda()
    Q = flat[1:].view(n, d)  # 4 bytes past a 16-byte boundary: scalar head
    od = torch.empty((n, k), device="cuda")
    oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
    go = lambda q, r: knn.search_device(q.data_ptr(), n, r.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr())
    go(Q, R)
    torch.cuda.synchronize()
    for (qi, qc) in [(0, 1), (100, 7), (n - 1, d - 1)]:
        Qb = Q.clone() if (qi, qc) != (0, 1) else Q
        saved = Qb[qi, qc].item()
        Qb[qi, qc] = float("nan")
        with pytest.raises(ValueError, match=rf"^PointSet: non-finite coordinate at point {qi}, dimension {qc}$"):
            go(Qb, R)
        Qb[qi, qc] = saved
    Rb = R.clone()
    Rb[m - 1, d - 1] = float("inf")
    with pytest.raises(ValueError, match=rf"^PointSet: non-finite coordinate at point {m - 1}, dimension {d - 1}$"):
        go(Q, Rb)
    go(Q, R)
    torch.cuda.synchronize()
    ri, _ = oracle.knn(Q[:20].cpu().numpy(), R.cpu().numpy(), k)
    assert (oi[:20].cpu().numpy() == ri).all()


@pytest.mark.gpu
def test_device_search_query_chunks(knn, oracle):
    """A device-pointer search over more queries than one tensor-path chunk
    (262144): rows on both sides of the chunk boundary are exact, and the
    fallback count is summed over the chunks (tie-saturated queries in each)."""
    import torch
    n, m, d, k = 300000, 20000, 16, 10
    R = oracle.uniform_f32(m, d, 45)
    R[:200] = 5.0  # 200 copies of one point far from the rest
    Q = oracle.uniform_f32(n, d, 46)
    Q[1000:1100] = R[0]  # their 200 tied neighbours overflow the fast path
    Q[280000:280100] = R[0]
    Qd, Rd = torch.from_numpy(Q).cuda(), torch.from_numpy(R).cuda()
    od = torch.empty((n, k), device="cuda")
    oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
    knn.search_device(Qd.data_ptr(), n, Rd.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(),
                      path=knn.PATH_TENSOR)
    torch.cuda.synchronize()
    assert knn.last_fallback_count() == 200
    rows = np.r_[0:64, 1000:1100:10, 262100:262200, 280000:280100:10, n - 64:n]
    te = knn.bf_knn(Q[rows], R, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (oi.cpu().numpy()[rows] == te.index).all()
    assert (od.cpu().numpy()[rows] == te.distance).all()


def test_pipelined_host_search(knn, oracle):
    """n >= 2 pipeline chunks: the one-shot host API overlaps query H2D / D2H
    with the search.  Results, device-side value checks and the deferred
    certification fallbacks behave as in the staged path."""
    n, m, d, k = 70000, 3000, 24, 10
    R = oracle.uniform_f32(m, d, 51)
    Q = oracle.uniform_f32(n, d, 52)
    t = knn.bf_knn(Q, R, k)
    te = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (t.index == te.index).all() and (t.distance == te.distance).all()
    Qb = Q.copy()
    Qb[53333, 5] = np.nan
    with pytest.raises(ValueError, match=r"^PointSet: non-finite coordinate at point 53333, dimension 5$"):
        knn.bf_knn(Qb, R, k)
    # a tie-saturated block of queries: uncertified, resolved after the pipeline
    Rd = R.copy()
    Rd[: 2000] = Rd[0]
    Qd = Q.copy()
    Qd[40000:40100] = Rd[0]
    td = knn.bf_knn(Qd, Rd, k)
    assert knn.last_fallback_count() > 0
    tde = knn.bf_knn(Qd, Rd, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (td.index == tde.index).all() and (td.distance == tde.distance).all()
