"""Dev tool (GPU): e2e breakdown of the host-API search on config B."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0804_1448_b200 as knn
n = m = 38400; d = 96; k = 20
Qd = torch.empty((n, d), device="cuda"); Rd = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(Qd.data_ptr(), n * d, 1); knn.fill_uniform_device(Rd.data_ptr(), m * d, 2)
Qh = torch.empty((n, d), pin_memory=True); Rh = torch.empty((m, d), pin_memory=True)
Qh.copy_(Qd.cpu()); Rh.copy_(Rd.cpu())
od = torch.empty((n, k), pin_memory=True); oi = torch.empty((n, k), dtype=torch.int64, pin_memory=True)
def tm(f, reps=10):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
h2d = tm(lambda: (Qd.copy_(Qh, non_blocking=True), Rd.copy_(Rh, non_blocking=True)))
ogd = torch.empty((n, k), device="cuda"); ogi = torch.empty((n, k), dtype=torch.int64, device="cuda")
d2h = tm(lambda: (od.copy_(ogd, non_blocking=True), oi.copy_(ogi, non_blocking=True)))
dev = tm(lambda: knn.search_device(Qd.data_ptr(), n, Rd.data_ptr(), m, d, k, ogd.data_ptr(), ogi.data_ptr()))
e2e = tm(lambda: knn.bf_knn(Qh.numpy(), Rh.numpy(), k, out=(od.numpy(), oi.numpy())))
print(f"H2D {h2d:.3f} ms ({(n+m)*d*4/h2d/1e6:.1f} GB/s)  D2H {d2h:.3f} ms ({n*k*12/d2h/1e6:.1f} GB/s)  device search {dev:.3f} ms  e2e {e2e:.3f} ms", flush=True)
