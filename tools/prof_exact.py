"""Dev tool (GPU): the exact SIMT path on config B (device-resident)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0804_1448_b200 as knn
n = m = int(sys.argv[1]) if len(sys.argv) > 1 else 38400
d = int(sys.argv[2]) if len(sys.argv) > 2 else 96
k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
metric = int(sys.argv[4]) if len(sys.argv) > 4 else 0
Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(Q.data_ptr(), n * d, 11); knn.fill_uniform_device(R.data_ptr(), m * d, 12)
od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
go = lambda: knn.search_device(Q.data_ptr(), n, R.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(), metric=metric, path=knn.PATH_EXACT)
go(); torch.cuda.synchronize()
knn.profile_enable(True); go(); torch.cuda.synchronize()
prof = knn.profile_collect(); knn.profile_enable(False)
print((n, m, d, k, metric), {kk: round(v[0] * 1e3, 1) for kk, v in prof.items()}, flush=True)
