"""bench.py's multi-GPU control flow on CPU (gloo, world_size 2): the real
run_line -- reference shards at their global counter offsets, the NCCL
unique-id broadcast, one communicator per rank, the rank-major all-gather +
(key, index) merge, the max-over-ranks timing, the roofline block, the JSON
line and the oracle correctness gate -- with only the device kernels replaced
by a host stub (the kernels themselves are covered by the GPU tests).  Also:
`bench.py --gpus N` without torchrun never silently measures one GPU."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class _Ev:
    t = 0.0


class _Clock:
    window = None

    def start(self):
        pass

    def stop(self):
        pass

    def summary(self):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["cpu stub"]}


class StubBackend:
    """bench.CudaBackend's interface on host tensors; searches by the oracle."""

    def __init__(self):
        from oracle.oracle import Oracle
        self.orc = Oracle()
        self.searches = 0

    def empty(self, shape, dtype="f32"):
        return torch.empty(shape, dtype=torch.float32 if dtype == "f32" else torch.int64)

    def fill_uniform(self, buf, seed, offset):
        out = np.empty(buf.numel(), np.float32)
        self.orc.lib.ko_fill_counter_f32(out, offset, buf.numel(), seed)
        buf.copy_(torch.from_numpy(out).view(buf.shape))

    def host(self, buf):
        return buf.numpy()

    def sync(self):
        pass

    def index(self, R, m, d, lo):
        class Ix:
            def close(self_):
                pass
        ix = Ix()
        ix.R, ix.m, ix.lo = R.numpy(), m, lo
        return ix

    def unique_id(self):
        return os.urandom(128)

    def comm(self, uid, world, rank):
        assert len(uid) == 128
        class C:
            def close(self_):
                pass
        c = C()
        c.world, c.rank = world, rank
        return c

    def _local(self, index, Q, k):
        self.searches += 1
        idx, dist_ = self.orc.knn(Q.numpy(), index.R, k)
        return dist_, idx + index.lo

    def search(self, index, Q, n, k, od, oi, path):
        d_, i_ = self._local(index, Q, k)
        od.copy_(torch.from_numpy(d_.astype(np.float32)))
        oi.copy_(torch.from_numpy(i_))

    def dist_search(self, comm, index, Q, n, k, od, oi, path):
        d_, i_ = self._local(index, Q, k)
        dk = [torch.empty((n, k), dtype=torch.float64) for _ in range(comm.world)]
        ik = [torch.empty((n, k), dtype=torch.int64) for _ in range(comm.world)]
        dist.all_gather(dk, torch.from_numpy(d_))
        dist.all_gather(ik, torch.from_numpy(i_))
        K = torch.stack(dk).numpy().transpose(1, 0, 2).reshape(n, -1)
        I = torch.stack(ik).numpy().transpose(1, 0, 2).reshape(n, -1)
        order = np.lexsort((I, K), axis=1)[:, :k]
        od.copy_(torch.from_numpy(np.take_along_axis(K, order, 1).astype(np.float32)))
        oi.copy_(torch.from_numpy(np.take_along_axis(I, order, 1)))

    def flush_l2(self):
        pass

    def event(self):
        return _Ev()

    def record(self, ev):
        import time
        ev.t = time.perf_counter()

    def elapsed_ms(self, a, b):
        return (b.t - a.t) * 1e3

    def profile_enable(self, on, only=""):
        pass

    def profile_collect(self):
        return {"tc_filter_kernel": (1.0, 2)}

    def reset_launch_count(self):
        self.searches = 0

    def launch_count(self):
        return self.searches

    def clocks(self):
        return _Clock()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    args = bench.parse(["--gpus", str(world), "--steps", "2", "--warmup", "1", "--config", "A"])
    plumb = bench.DistPlumbing(world, rank, "gloo")
    be = StubBackend()
    line = bench.run_line(be, plumb, "A", cfg, args, world, rank, 0)
    if rank == 0:
        out["line"] = json.dumps(line)
    dist.destroy_process_group()


def test_bench_reference_sharded_flow_world2():
    cfg = dict(m=3000, n=200, d=16, k=20)
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(2, _port(), cfg, out), nprocs=2, join=True)
        line = json.loads(out["line"])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["parallelism"].startswith("reference-sharded x2")
    assert line["correctness_gate"]["result"] == "pass"
    assert line["roofline"]["bound"] == "tensor" and line["roofline"]["launches"] == 2
    assert line["gpu_launches"] == 2  # the two timed steps, one local search each
    assert line["e2e"] is None  # no device: the host-buffer leg needs the real engine


def test_bench_gpus_without_torchrun_never_runs_one_gpu():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    msg = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" in msg and msg["n_gpus"] == 2
