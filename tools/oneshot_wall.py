"""Dev tool (GPU): wall-clock per call of the one-shot device search
(knn_b200_search_device) on the default stream and on torch's stream."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0804_1448_b200 as knn
n = m = 38400; d = 96; k = 20
Q = torch.empty((n, d), device="cuda"); R = torch.empty((m, d), device="cuda")
knn.fill_uniform_device(Q.data_ptr(), n * d, 1); knn.fill_uniform_device(R.data_ptr(), m * d, 2)
od = torch.empty((n, k), device="cuda"); oi = torch.empty((n, k), dtype=torch.int64, device="cuda")
ns = torch.cuda.Stream()
for name, s in (("stream 0 (synchronous API)", 0), ("own stream", ns.cuda_stream)):
    go = lambda: knn.search_device(Q.data_ptr(), n, R.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(), stream=s)
    for _ in range(3): go()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); go(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    print(name, "ms per call (wall, synced):", [round(t, 3) for t in ts], flush=True)
# host enqueue time with the GPU busy (the host runs ahead), one-shot vs index
s = ns.cuda_stream
busy = torch.empty(1 << 29, dtype=torch.uint8, device="cuda")
ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
calls = {
    "one-shot": lambda: knn.search_device(Q.data_ptr(), n, R.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(), stream=s),
    "index": lambda: ix.search_device(Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(), stream=s),
}
for name, go in calls.items():
    ts = []
    for _ in range(8):
        with torch.cuda.stream(ns):
            for _ in range(6): busy.zero_()
        t0 = time.perf_counter(); go(); ts.append((time.perf_counter() - t0) * 1e3)
        torch.cuda.synchronize()
    print(name, "host enqueue ms (GPU busy):", [round(t, 3) for t in ts], flush=True)
# Python-side costs
t0 = time.perf_counter()
for _ in range(100): o = knn._opts(knn.BfConfig(path=knn.PATH_AUTO), stream=s)
print("_opts us:", round((time.perf_counter() - t0) * 1e4, 2), flush=True)
