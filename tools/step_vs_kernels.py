"""Dev tool (GPU): bench-style timed steps (L2 flush between) vs the engine's
per-kernel event times, step by step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0804_1448_b200 as knn
n = m = 38400; d = 96; k = 20
Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(Q.data_ptr(), n * d, 1); knn.fill_uniform_device(R.data_ptr(), m * d, 2)
od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
stream = torch.cuda.current_stream()
s = stream.cuda_stream
go = lambda: ix.search_device(Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(), stream=s)
for _ in range(3): go()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
for mode in ("noflush", "flush", "flush+clean"):
    for i in range(4):
        if mode != "noflush": flush.zero_()
        if mode == "flush+clean": clean.sum()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        knn.profile_enable(True)
        a.record(stream); go(); b.record(stream)
        torch.cuda.synchronize()
        knn.profile_enable(False)
        prof = knn.profile_collect()
        ks = {kk: round(v[0] * 1e3, 1) for kk, v in prof.items()}
        print(mode, "step us", round(a.elapsed_time(b) * 1e3, 1), "kernels", ks, "sum", round(sum(ks.values()), 1), flush=True)
