"""Dev tool (GPU): per-kernel device times for one shape (tensor path)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0804_1448_b200 as knn
n, m, d, k = [int(x) for x in sys.argv[1:5]]
Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(Q.data_ptr(), n * d, 11); knn.fill_uniform_device(R.data_ptr(), m * d, 12)
od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
go = lambda: knn.search_device(Q.data_ptr(), n, R.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(), path=knn.PATH_AUTO)
go(); torch.cuda.synchronize()
knn.profile_enable(True); go(); torch.cuda.synchronize()
prof = knn.profile_collect(); knn.profile_enable(False)
print((n, m, d, k), "fallbacks", knn.last_fallback_count(), {kk: round(v[0] * 1e3, 1) for kk, v in prof.items()}, flush=True)
