"""Dev tool (GPU): one config-E shard (m = 10M/8 = 1.25M references, n = 100K
queries, d = 128, k = 20) -- device-resident timing + oracle check of a sample."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0804_1448_b200 as knn
from oracle.oracle import Oracle, compare
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1250000
n, d, k = 100000, 128, 20
Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(R.data_ptr(), m * d, 77); knn.fill_uniform_device(Q.data_ptr(), n * d, 78)
od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
go = lambda: knn.search_device(Q.data_ptr(), n, R.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(), path=knn.PATH_AUTO)
go(); torch.cuda.synchronize()
knn.profile_enable(True)
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); go(); e.record(); torch.cuda.synchronize()
prof = knn.profile_collect(); knn.profile_enable(False)
ms = s.elapsed_time(e)
print(f"m={m} n={n} d={d} k={k}: {ms:.2f} ms  {n / ms * 1e3 / 1e6:.2f} M q/s  fallbacks={knn.last_fallback_count()}",
      {kk: round(v[0], 2) for kk, v in prof.items()}, flush=True)
o = Oracle()
sel = np.random.default_rng(1).choice(n, 64, replace=False)
Rh = R.cpu().numpy(); Qh = Q.cpu().numpy()[sel]
ri, rd = o.knn(Qh, Rh, k)
print(compare(oi.cpu().numpy()[sel], od.cpu().numpy()[sel], ri, rd, Qh, Rh, oracle=o), flush=True)
