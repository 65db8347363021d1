"""Dev tool (GPU): host-side enqueue time of one device-resident search (index
handle), vs its device time."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0804_1448_b200 as knn
n = m = 38400; d = 96; k = 20
Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(Q.data_ptr(), n * d, 1); knn.fill_uniform_device(R.data_ptr(), m * d, 2)
od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
s = torch.cuda.current_stream().cuda_stream
go = lambda: ix.search_device(Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(), stream=s)
for _ in range(3): go()
torch.cuda.synchronize()
busy = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    busy.zero_(); busy.zero_(); busy.zero_()  # keep the GPU busy while the host enqueues
    t0 = time.perf_counter(); go(); ts.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
print("host enqueue us per search:", [round(t, 1) for t in ts])
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
busy.zero_(); busy.zero_(); busy.zero_()
e0.record(); go(); e1.record(); torch.cuda.synchronize()
print("device time with host ahead (us):", round(e0.elapsed_time(e1) * 1e3, 1))
torch.cuda.synchronize()
e0.record(); go(); e1.record(); torch.cuda.synchronize()
print("device time, host not ahead (us):", round(e0.elapsed_time(e1) * 1e3, 1))
