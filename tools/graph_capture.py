"""Dev tool (GPU): capture an index search (caller stream, small k) into a
CUDA graph and replay it; compare with the eager result and time both."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0804_1448_b200 as knn
n = m = 38400; d = 96; k = 20
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(Q.data_ptr(), n * d, 1, 0, s.cuda_stream); knn.fill_uniform_device(R.data_ptr(), m * d, 2, 0, s.cuda_stream)
od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
go = lambda: ix.search_device(Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
for _ in range(3): go()
torch.cuda.synchronize()
ref_i = oi.clone(); ref_d = od.clone()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    go()
od.zero_(); oi.zero_()
g.replay(); torch.cuda.synchronize()
print("graph replay identical:", bool((oi == ref_i).all() and (od == ref_d).all()), flush=True)
for name, f in (("eager", go), ("graph", g.replay)):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    f(); torch.cuda.synchronize()
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    print(name, "us per search", round(e0.elapsed_time(e1) / 20 * 1e3, 1), flush=True)
