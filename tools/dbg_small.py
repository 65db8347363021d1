import sys, os, time
sys.path.insert(0, '.')
import numpy as np
import paper_0804_1448_b200 as knn
from oracle.oracle import Oracle, compare
o = Oracle()
for (n, m, d, k) in [(256, 128, 32, 4), (256, 1024, 32, 20), (300, 2000, 32, 20), (1000, 5000, 96, 20)]:
    R = o.uniform_f32(m, d, 1); Q = o.uniform_f32(n, d, 2)
    print("start", (n, m, d, k), flush=True)
    t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    ri, rd = o.knn(Q, R, k)
    print((n, m, d, k), compare(t.index, t.distance, ri, rd, Q, R, oracle=o), knn.last_fallback_count(), flush=True)
