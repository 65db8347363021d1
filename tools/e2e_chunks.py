"""Dev tool (GPU): host-API e2e time on config B for several pipeline chunk
sizes (E2E_SHAPE="n,m,d", E2E_CHUNKS="a,b,..."; KNN_B200_PIPE_CHUNK is read once per process, so each size runs in its
own subprocess; two interleaved rounds)."""
import os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if os.environ.get("_E2E_CHILD"):
    sys.path.insert(0, ROOT)
    import torch
    import paper_0804_1448_b200 as knn
    n, m, d = (int(x) for x in os.environ.get("E2E_SHAPE", "38400,38400,96").split(","))
    k = 20
    Qh = torch.rand((n, d)).pin_memory(); Rh = torch.rand((m, d)).pin_memory()
    od = torch.empty((n, k), pin_memory=True); oi = torch.empty((n, k), dtype=torch.int64, pin_memory=True)
    f = lambda: knn.bf_knn(Qh.numpy(), Rh.numpy(), k, out=(od.numpy(), oi.numpy()))
    for _ in range(3): f()
    ts = []
    for _ in range(15):
        t0 = time.perf_counter(); f(); ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    print((n, m, d), os.environ.get("KNN_B200_PIPE_CHUNK"), "median ms", round(ts[len(ts) // 2], 3), "min", round(ts[0], 3), flush=True)
else:
    for rep in range(2):
        for c in os.environ.get("E2E_CHUNKS", "65536,32768,12800,9600,6400").split(","):
            env = dict(os.environ, _E2E_CHILD="1", KNN_B200_PIPE_CHUNK=c)
            subprocess.run([sys.executable, __file__], env=env)
