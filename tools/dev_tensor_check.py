import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_0804_1448_b200 as knn
from oracle.oracle import Oracle, compare
o = Oracle()
for (n, m, d, k) in [(300, 2000, 32, 20), (1000, 5000, 96, 20), (128, 128, 8, 1), (4800, 4800, 32, 20), (2000, 38400, 96, 20), (700, 9000, 128, 10), (257, 1000, 64, 16)]:
    R = o.uniform_f32(m, d, 1 + d); Q = o.uniform_f32(n, d, 2 + d)
    ri, rd = o.knn(Q, R, k)
    t0 = time.time()
    t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    dt = time.time() - t0
    rep = compare(t.index, t.distance, ri, rd, Q, R, oracle=o)
    te = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    same = (te.index == t.index).all() and (te.distance == t.distance).all()
    print((n, m, d, k), rep, 'fallbacks', knn.last_fallback_count(), 'bitwise_eq_exact', same, f'{dt:.3f}s', flush=True)
