"""Dev tool (GPU): every k in 1..40 and a few large k on one moderate shape --
tensor path vs exact path bitwise on a query sample, fallback counts."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_0804_1448_b200 as knn
rng = np.random.default_rng(3)
m, n, d = 20000, 2048, 29
R = rng.random((m, d), dtype=np.float32)
Q = rng.random((n, d), dtype=np.float32)
rows = np.arange(0, n, 32)
bad = []
for k in list(range(1, 41)) + [64, 100, 129, 256, 500, 1024]:
    t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    fb = knn.last_fallback_count()
    te = knn.bf_knn(Q[rows], R, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    ok = (t.index[rows] == te.index).all() and (t.distance[rows] == te.distance).all()
    print(f"k={k} fallbacks={fb} bitwise={'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        bad.append(k)
print("mismatches:", bad)
