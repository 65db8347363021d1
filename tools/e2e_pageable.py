"""Dev tool (GPU): host-API e2e on config B with pageable (numpy) vs pinned host buffers."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0804_1448_b200 as knn
n = m = 38400; d = 96; k = 20
rng = np.random.default_rng(1)
Qp = rng.random((n, d), dtype=np.float32); Rp = rng.random((m, d), dtype=np.float32)
odp = np.empty((n, k), np.float32); oip = np.empty((n, k), np.int64)
Qh = torch.from_numpy(Qp).pin_memory(); Rh = torch.from_numpy(Rp).pin_memory()
od = torch.empty((n, k), pin_memory=True); oi = torch.empty((n, k), dtype=torch.int64, pin_memory=True)
for name, f in (("pinned", lambda: knn.bf_knn(Qh.numpy(), Rh.numpy(), k, out=(od.numpy(), oi.numpy()))),
                ("pageable", lambda: knn.bf_knn(Qp, Rp, k, out=(odp, oip)))):
    for _ in range(3): f()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); f(); ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    print(f"{name}: median {ts[5]:.3f} ms -> {n / ts[5] / 1e3:.1f} M q/s", flush=True)
