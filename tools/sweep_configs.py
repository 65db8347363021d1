"""Dev tool (GPU): device-resident search time for the BASELINE configs C
(d sweep, m=n=19200, k=20) and D (k sweep, m=n=38400, d=64), auto path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0804_1448_b200 as knn

def run(n, m, d, k, reps=3, path=None):
    path = knn.PATH_AUTO if path is None else path
    Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
    knn.fill_uniform_device(Q.data_ptr(), n * d, 11); knn.fill_uniform_device(R.data_ptr(), m * d, 12)
    od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
    go = lambda: knn.search_device(Q.data_ptr(), n, R.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(), path=path)
    go(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): go()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"n={n} m={m} d={d} k={k} path={path}: {ms:.3f} ms  {n / ms * 1e3 / 1e6:.2f} M q/s  fallbacks={knn.last_fallback_count()}", flush=True)

which = sys.argv[1] if len(sys.argv) > 1 else "CD"
if "C" in which:
    for d in (8, 16, 32, 64, 80, 96, 128):
        run(19200, 19200, d, 20)
if "D" in which:
    for k in (1, 20, 100, 256, 1024):
        run(38400, 38400, 64, k, reps=1 if k > 32 else 3)
