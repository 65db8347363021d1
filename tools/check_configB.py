"""Dev tool (GPU): tensor path on config B (m=n=38400, d=96, k=20) checked
against the oracle on a query subsample."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_0804_1448_b200 as knn
from oracle.oracle import Oracle, compare
o = Oracle()
n = m = int(sys.argv[1]) if len(sys.argv) > 1 else 38400
d = int(sys.argv[2]) if len(sys.argv) > 2 else 96
k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
R = o.uniform_f32(m, d, 7); Q = o.uniform_f32(n, d, 8)
t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
fb = knn.last_fallback_count()
sel = np.random.default_rng(0).choice(n, 256, replace=False)
ri, rd = o.knn(Q[sel], R, k)
print((n, m, d, k), "fallbacks", fb, compare(t.index[sel], t.distance[sel], ri, rd, Q[sel], R, oracle=o), flush=True)
