"""Dev tool (GPU): large-k tensor path vs oracle on moderate shapes + timing."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_0804_1448_b200 as knn
from oracle.oracle import Oracle, compare
o = Oracle()
for (n, m, d, k) in [(300, 2000, 32, 40), (500, 6000, 64, 100), (400, 20000, 64, 256), (256, 38400, 64, 1024), (300, 5000, 128, 33)]:
    R = o.uniform_f32(m, d, 3); Q = o.uniform_f32(n, d, 4)
    t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    fb = knn.last_fallback_count()
    ri, rd = o.knn(Q, R, k)
    print((n, m, d, k), compare(t.index, t.distance, ri, rd, Q, R, oracle=o), "fallbacks", fb, flush=True)
