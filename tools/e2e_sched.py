"""Dev tool (GPU): e2e (host API, pinned buffers) of config B under the
pipelined host search's chunk schedule given by KNN_B200_PIPE_CHUNKS."""
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
f = lambda: knn.bf_knn(Qh.numpy(), Rh.numpy(), k, out=(od.numpy(), oi.numpy()))
for _ in range(3): f()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
ts.sort()
print(f"chunks={os.environ.get('KNN_B200_PIPE_CHUNKS', 'default')} e2e median {ts[10]*1e3:.3f} ms "
      f"min {ts[0]*1e3:.3f} ms -> {n / ts[10] / 1e6:.1f} M q/s", flush=True)
