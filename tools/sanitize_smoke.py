"""Dev tool (GPU, under compute-sanitizer): small searches over every kernel
family -- exact (3 metrics, list variants, stream-K slots), tensor small/large
k, device fallback, Mahalanobis whitening, merge."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_0804_1448_b200 as knn
rng = np.random.default_rng(5)
def run(n, m, d, k, metric=knn.EUCLIDEAN, path=knn.PATH_AUTO, R=None):
    Q = rng.random((n, d), dtype=np.float32)
    R = rng.random((m, d), dtype=np.float32) if R is None else R
    t = knn.bf_knn(Q, R, k, knn.Metric(metric), config=knn.BfConfig(path=path))
    assert (t.index >= 0).all()
for metric in (knn.EUCLIDEAN, knn.MANHATTAN, knn.CHEBYSHEV):
    for k in (1, 33, 129, 300):
        run(150, 3000, 37, k, metric, knn.PATH_EXACT)
run(300, 5000, 24, 20, path=knn.PATH_TENSOR)
run(300, 5000, 24, 100, path=knn.PATH_TENSOR)
run(200, 3000, 96, 1024, path=knn.PATH_TENSOR)
dup = np.repeat(rng.random((1, 16), dtype=np.float32), 9000, axis=0)
run(50, 9000, 16, 20, path=knn.PATH_TENSOR, R=dup)
# round 2: narrow folded-norm K blocks (d = 64, 128), the large-k device
# fallback (k = 64: exact lists from a query list; k = 300: the exact path's
# threshold-log selection over a query list), the exact path's large-k
# selection (L1 / L2 with d > 128) and its forced list-path fallback
run(300, 5000, 128, 20, path=knn.PATH_TENSOR)
run(600, 20000, 29, 28, path=knn.PATH_TENSOR)  # 32-entry bound lists, several units per CTA
run(300, 5000, 64, 150, path=knn.PATH_TENSOR)
run(50, 9000, 16, 64, path=knn.PATH_TENSOR, R=dup)
run(50, 9000, 16, 300, path=knn.PATH_TENSOR, R=dup)
run(150, 6000, 24, 300, knn.MANHATTAN, knn.PATH_EXACT)
run(150, 6000, 160, 200, knn.EUCLIDEAN, knn.PATH_EXACT)
far = rng.random((8192, 8), dtype=np.float32) + 50.0
far[::28] = rng.random((len(far[::28]), 8), dtype=np.float32) * 0.1
Qn = rng.random((40, 8), dtype=np.float32) * 0.1
knn.bf_knn(Qn, far, 300, knn.Metric(knn.MANHATTAN), config=knn.BfConfig(path=knn.PATH_EXACT))
M = np.eye(8) * 2.0
Q = rng.random((40, 8), dtype=np.float32); R = rng.random((900, 8), dtype=np.float32)
knn.bf_knn(Q, R, 5, knn.Metric.mahalanobis(8, M.ravel()))
print("sanitize smoke ok", flush=True)
