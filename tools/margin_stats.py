"""Dev tool: distribution of (candidates within the certified bound) - k on the
BASELINE configs, to size the candidate list K' = k + extra (set
KNN_B200_DEBUG_HIST=1; the engine prints a histogram per tensor-path search)."""
import os, sys
os.environ["KNN_B200_DEBUG_HIST"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_0804_1448_b200 as knn

def uni(rows, d, seed):
    import torch
    x = torch.empty((rows, d), dtype=torch.float32, device="cuda")
    knn.fill_uniform_device(x.data_ptr(), rows * d, seed)
    torch.cuda.synchronize()
    return x.cpu().numpy()

for (n, m, d, k) in [(38400, 38400, 96, 20), (19200, 19200, 8, 20), (19200, 19200, 32, 20),
                     (19200, 19200, 64, 20), (19200, 19200, 128, 20), (4800, 4800, 32, 20),
                     (38400, 38400, 64, 1), (20000, 200000, 128, 20)]:
    Q, R = uni(n, d, 1 + d), uni(m, d, 2 + d)
    knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    print((n, m, d, k), "fallbacks", knn.last_fallback_count(), flush=True)
