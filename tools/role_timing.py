"""Dev tool: per-role cycle accounting of the tcgen05 filter kernel
(KNN_B200_DEBUG_ROLES=1) on the headline config."""
import os, sys
os.environ["KNN_B200_DEBUG_ROLES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0804_1448_b200 as knn
n = m = int(sys.argv[1]) if len(sys.argv) > 1 else 38400
d = int(sys.argv[2]) if len(sys.argv) > 2 else 96
k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(Q.data_ptr(), n * d, 1); knn.fill_uniform_device(R.data_ptr(), m * d, 2)
od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
for _ in range(3):
    knn.search_device(Q.data_ptr(), n, R.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(), path=knn.PATH_TENSOR)
torch.cuda.synchronize()
