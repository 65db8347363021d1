"""GPU tests of the exact path's large-k threshold-log selection
(csrc/exact_large.cu: sample threshold, threshold-log pass, block select,
list-path fallback) for 128 < k <= 1024 on the metrics the tensor path does not
serve (L1, L-inf, L2 with d > 128): against the oracle with the north-star
comparator, and bitwise against the list path it replaces (the same exact FP32
keys and (key, index) order; KNN_B200_EXACT_LARGE=0 selects the list path in a
subprocess).  Reference semantics: src/topk.cpp:17-33 (k smallest, ties by
ascending index), include/knn/metric.hpp:22-44 (the keys)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle.oracle import CHEBYSHEV, EUCLIDEAN, MANHATTAN, compare

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def list_path_result(Q, R, k, metric, tmp_path):
    """The same search on the list path, in a subprocess (the switch is read once)."""
    src = tmp_path / "in.npz"
    out = tmp_path / "out.npz"
    np.savez(src, Q=Q, R=R)
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_0804_1448_b200 as knn\n"
        "z = np.load(%r)\n"
        "t = knn.bf_knn(z['Q'], z['R'], %d, knn.Metric(%d), config=knn.BfConfig(path=knn.PATH_EXACT, device=0))\n"
        "np.savez(%r, idx=t.index, dist=t.distance)\n" % (ROOT, str(src), k, metric, str(out)))
    env = dict(os.environ, KNN_B200_EXACT_LARGE="0")
    subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=600)
    z = np.load(out)
    return z["idx"], z["dist"]


def exact(knn, Q, R, k, metric):
    return knn.bf_knn(Q, R, k, knn.Metric(metric), config=knn.BfConfig(path=knn.PATH_EXACT, device=0))


@pytest.mark.parametrize("metric,d", [(MANHATTAN, 24), (CHEBYSHEV, 16), (EUCLIDEAN, 160)])
@pytest.mark.parametrize("k", [129, 300, 1024])
def test_large_k_vs_oracle(knn, oracle, metric, d, k):
    n, m = 160, 9000
    Q = oracle.uniform_f32(n, d, 901 + k)
    R = oracle.uniform_f32(m, d, 902 + k)
    ri, rd = oracle.knn(Q, R, k, metric)
    t = exact(knn, Q, R, k, metric)
    rep = compare(t.index, t.distance, ri, rd, Q, R, metric, oracle=oracle)
    assert rep.ok, f"k={k} metric={metric}: {rep}"
    assert knn.last_fallback_count() == 0


@pytest.mark.parametrize("metric", [MANHATTAN, EUCLIDEAN])
def test_large_k_bitwise_equals_list_path(knn, oracle, metric, tmp_path):
    # ragged shapes: partial last tile, several CTAs per query block, odd d
    n, m, d, k = 300, 12345, 33 if metric == MANHATTAN else 131, 400
    Q = oracle.uniform_f32(n, d, 911) * 4 - 2
    R = oracle.uniform_f32(m, d, 912) * 4 - 2
    t = exact(knn, Q, R, k, metric)
    li, ld = list_path_result(Q, R, k, metric, tmp_path)
    assert (t.index == li).all()
    assert (t.distance == ld).all()


def test_large_k_ties_resolve_by_index(knn, oracle, tmp_path):
    """Dense exact ties at the k-th key: integer grid points, many duplicates;
    the kept tie entries must be the lowest indices (topk.cpp:11-15)."""
    rng = np.random.default_rng(5)
    n, m, d, k = 130, 8192, 4, 500
    R = rng.integers(0, 3, size=(m, d)).astype(np.float32)
    Q = rng.integers(0, 3, size=(n, d)).astype(np.float32)
    for metric in (MANHATTAN, CHEBYSHEV):
        t = exact(knn, Q, R, k, metric)
        li, ld = list_path_result(Q, R, k, metric, tmp_path)
        assert (t.index == li).all(), metric
        assert (t.distance == ld).all(), metric
        ri, rd = oracle.knn(Q, R, k, metric)
        assert (t.index == ri).all(), metric


def test_large_k_unrepresentative_sample_falls_back(knn, oracle):
    """Every sampled reference (rows 0, s, 2s, ...) sits next to the queries and
    the rest far away: the sample threshold admits fewer than k keys, the
    certificate fails and the list path answers those queries."""
    n, m, d, k = 40, 8192, 8, 300
    stride = (3 * k) // 32
    R = oracle.uniform_f32(m, d, 921) + 50.0
    R[::stride] = oracle.uniform_f32(len(R[::stride]), d, 922) * 0.1
    Q = oracle.uniform_f32(n, d, 923) * 0.1
    for metric in (MANHATTAN, EUCLIDEAN):
        t = knn.bf_knn(Q, R, k, knn.Metric(metric), config=knn.BfConfig(path=knn.PATH_EXACT, device=0))
        assert knn.last_fallback_count() == n
        ri, rd = oracle.knn(Q, R, k, metric)
        rep = compare(t.index, t.distance, ri, rd, Q, R, metric, oracle=oracle)
        assert rep.ok, str(rep)


def test_large_k_query_chunks(knn, oracle):
    """More than one 32768-query chunk: every chunk's rows land in place, the
    fallback count sums over the chunks."""
    n, m, d, k = 33000, 4096, 8, 150
    Q = oracle.uniform_f32(n, d, 931)
    R = oracle.uniform_f32(m, d, 932)
    t = exact(knn, Q, R, k, MANHATTAN)
    assert knn.last_fallback_count() == 0
    rows = np.r_[0:40, 32750:32800, n - 40:n]
    ri, rd = oracle.knn(Q[rows], R, k, MANHATTAN)
    rep = compare(t.index[rows], t.distance[rows], ri, rd, Q[rows], R, MANHATTAN, oracle=oracle)
    assert rep.ok, str(rep)
