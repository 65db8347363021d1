"""Dev tool (GPU): bench-style step time (index search on a side stream, L2
flush between steps) with and without the per-kernel profiling events."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0804_1448_b200 as knn
torch.cuda.set_stream(torch.cuda.Stream())
stream = torch.cuda.current_stream()
n = m = 38400; d = 96; k = 20
Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(Q.data_ptr(), n * d, 1, 0, stream.cuda_stream); knn.fill_uniform_device(R.data_ptr(), m * d, 2, 0, stream.cuda_stream)
od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
go = lambda: ix.search_device(Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(), stream=stream.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); clean = torch.ones(64 << 20, device="cuda")
for _ in range(3): go()
torch.cuda.synchronize()
for prof in (False, True, False, True):
    ts = []
    for _ in range(10):
        flush.zero_(); clean.sum()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        knn.profile_enable(prof)
        a.record(stream); go(); b.record(stream)
        knn.profile_enable(False)
    torch.cuda.synchronize()
    if prof: knn.profile_collect()
    print("profiling" if prof else "plain    ", "step us", round(a.elapsed_time(b) * 1e3, 1), flush=True)
