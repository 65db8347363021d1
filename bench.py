#!/usr/bin/env python3
"""Benchmark: kNN queries/s on BASELINE.json's configs (default: configs[1],
m = n = 38400, d = 96, k = 20, on 1 GPU; configs[4] -- m = 10M references,
n = 100K queries, d = 128, k = 20, reference-sharded -- on N > 1 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config A|B|C|D|E] [--path auto|exact|tensor]

ours (default)
    A "step" is one full search of all n queries against the reference set,
    inputs already resident in HBM.  N = 1: one device search through a
    device-resident index.  N > 1 (one rank per GPU, launched by torchrun -- or
    by this script itself when --gpus N > 1 is given without torchrun): rank r
    holds the contiguous reference rows shard_bounds(m, N, r) and all queries;
    each step is knn_b200_dist_search_device: the local shard search, an NCCL
    all-gather of the raw-key lists over the library's own communicator, and
    the device merge -- every rank ends with the full table.
    Total work is fixed, so scaling is "strong".
    Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA
    events on the launch stream with an L2 flush (256 MiB write, then a
    256 MiB read that evicts the dirty lines) between steps; barrier +
    synchronize around the timed region; max over ranks.
    e2e: the same metric through the public host API with host buffers and the
    copies inside the timed region (N = 1: knn_b200_search, the bf_knn drop-in,
    pinned buffers; N > 1: per rank the H2D of its reference shard and the
    queries, index creation, the distributed search, D2H of the table on
    rank 0).
    roofline: the dominant kernel's per-launch time from CUDA events around
    each of its launches on its stream inside the timed region, against
    MEASURED_PEAKS.json (tensor TF/s by 2 n m d for the tcgen05 filter; HBM
    GB/s by algorithmic bytes otherwise; low-d and large-k lines also carry
    candidate visits/s against the SM issue capacity).
    correctness gate: an oracle check of a query sample of the table the timed
    steps produced; no line is printed if it fails.
    cpu_baseline (rank 0, N = 1): the reference's own bf_knn (oracle/_ref), all
    host threads, on a bounded query sample of the same inputs.

reference (--impl reference)
    Rank 0 only: the reference's CPU bf_knn on the box's host cores, each step
    a bounded query sample of the same workload; other ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_B_QPS = 38400 / 43.74  # BF-CUDA 43.74 s on a GeForce 8800 GTX
METRIC = "kNN queries/sec (m=n=38400, d=96, k=20) at 1/2/4/8 B200 vs CPU ref"

# BASELINE.json "configs" (index, workloads)
CONFIGS = {
    "A": (0, [dict(m=4800, n=4800, d=32, k=20)]),
    "B": (1, [dict(m=38400, n=38400, d=96, k=20)]),
    "C": (2, [dict(m=19200, n=19200, d=dd, k=20) for dd in (8, 16, 32, 64, 80, 96, 128)]),
    "D": (3, [dict(m=38400, n=38400, d=64, k=kk) for kk in (1, 20, 100, 256, 1024)]),
    "E": (4, [dict(m=10_000_000, n=100_000, d=128, k=20)]),
}
# SM issue capacity: 148 SMs x 4 warp schedulers x 32 lanes x 1.965 GHz
ISSUE_THREAD_INST_PER_S = 148 * 4 * 32 * 1.965e9
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def derive_seed(master: int, a: int, b: int = 0, c: int = 0) -> int:
    """rng.hpp:17-28 (splitmix64 mixing), used for the bench's input seeds."""
    M = (1 << 64) - 1

    def step(state):
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return state, z ^ (z >> 31)

    st, out = step(master)
    st ^= (a * 0x9E3779B97F4A7C15) & M
    st, v = step(st)
    out ^= v
    st ^= (b * 0xBF58476D1CE4E5B9) & M
    st, v = step(st)
    out ^= v
    st ^= (c * 0x94D049BB133111EB) & M
    st, v = step(st)
    return out ^ v


def seeds(cfg):
    return (derive_seed(42, cfg["m"], cfg["d"], 0), derive_seed(42, cfg["n"], cfg["d"], 1))


def workload_name(letter, cfg):
    idx = CONFIGS[letter][0]
    return (f"configs[{idx}]: m={cfg['m']}, n={cfg['n']}, d={cfg['d']}, k={cfg['k']}, euclidean")


def shard_bounds(m, world, rank):
    from paper_0804_1448_b200.sharding import shard_bounds as sb
    return sb(m, world, rank)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


class ClockSampler:
    """NVML SM clock + throttle-reason sampler (runs in a thread)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples = []
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self._stop = threading.Event()
        self._t = None
        self.window = None

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        lo, hi = self.window or (self.samples[0][0], self.samples[-1][0])
        inside = [s for s in self.samples if lo <= s[0] <= hi] or self.samples
        reasons = set()
        for _, _, rs in inside:
            for bit, name in self.REASONS.items():
                if rs & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[1] for s in inside), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(inside)}


def measured_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, from
    the newest committed ncu --set full summary (profiles/r*_traffic.json)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    if not files:
        return None
    try:
        with open(files[-1]) as f:
            table = json.load(f)
    except Exception:
        return None
    key = kernel.replace("tc_", "").replace("_glist", "")
    for name, val in table.items():
        if key in name:
            return {"bytes_per_launch": int(val), "source": os.path.relpath(files[-1], ROOT)}
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ backends --
class CudaBackend:
    """The product path: device buffers from torch, every search through the
    engine's C ABI (paper_0804_1448_b200)."""

    def __init__(self, local: int):
        import torch

        import paper_0804_1448_b200 as knn
        self.torch, self.knn = torch, knn
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        self.local = local
        # a dedicated (non-default) stream: the engine, the L2 flush and the
        # step events all order on it (handle 0 would mean "engine stream")
        torch.cuda.set_stream(torch.cuda.Stream(self.dev))
        self.stream = torch.cuda.current_stream(self.dev)
        self.sptr = self.stream.cuda_stream
        self._flush = None

    # buffers
    def empty(self, shape, dtype="f32"):
        dt = {"f32": self.torch.float32, "i64": self.torch.int64}[dtype]
        return self.torch.empty(shape, dtype=dt, device=self.dev)

    def fill_uniform(self, buf, seed, offset):
        self.knn.fill_uniform_device(buf.data_ptr(), buf.numel(), seed, offset, self.sptr)

    def host(self, buf):
        return buf.cpu().numpy()

    def sync(self):
        self.torch.cuda.synchronize(self.dev)

    # engine objects
    def index(self, R, m, d, lo):
        return self.knn.Index(device_ptr=R.data_ptr(), m=m, d=d, index_base=lo, device=self.local)

    def unique_id(self):
        return self.knn.nccl_unique_id()

    def comm(self, uid, world, rank):
        return self.knn.Comm(uid, world, rank, self.local)

    def search(self, index, Q, n, k, od, oi, path):
        index.search_device(Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(), path=path,
                            stream=self.sptr)

    def search_oneshot(self, R, m, Q, n, d, k, od, oi, path):
        """bf_knn semantics on device buffers: the reference set prepared
        inside the call (no index handle)."""
        self.knn.search_device(Q.data_ptr(), n, R.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(),
                               path=path, stream=self.sptr, device=self.local)

    def dist_search(self, comm, index, Q, n, k, od, oi, path):
        comm.search_device(index, Q.data_ptr(), n, k, od.data_ptr(), oi.data_ptr(), path=path,
                           stream=self.sptr)

    # timing
    def flush_l2(self):
        if self._flush is None:
            self._flush = self.torch.empty(256 << 20, dtype=self.torch.uint8, device=self.dev)
            # a second buffer read after the flush write evicts the flush's dirty
            # lines, so their write-back lands before the step's start event
            self._clean = self.torch.ones(64 << 20, dtype=self.torch.float32, device=self.dev)
        self._flush.zero_()
        self._clean.sum()

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)

    def record(self, ev):
        ev.record(self.stream)

    def elapsed_ms(self, a, b):
        return a.elapsed_time(b)

    def profile_enable(self, on, only=""):
        self.knn.profile_enable(on, only=only)

    def profile_collect(self):
        return self.knn.profile_collect()

    def reset_launch_count(self):
        self.knn.reset_launch_count()

    def launch_count(self):
        return self.knn.launch_count()

    def clocks(self):
        return ClockSampler(self.local)


class DistPlumbing:
    """Rank-to-rank plumbing over torch.distributed (NCCL for GPUs, gloo in the
    CPU tests): the NCCL unique-id broadcast, barriers, max over ranks."""

    def __init__(self, world, rank, backend_name):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.world, self.rank = torch, dist, world, rank
        self.backend_name = backend_name

    def broadcast_bytes(self, b):
        obj = [b if self.rank == 0 else None]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def barrier(self):
        self.dist.barrier()

    def max(self, x: float) -> float:
        t = self.torch.tensor([x], dtype=self.torch.float64)
        if self.backend_name == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


# ------------------------------------------------------------------ our arm --
def dominant_roofline(name, per_launch_ms, launches, cfg, m_local, world, peaks, peak_src):
    """Roofline of the dominant kernel: its algorithmic work per launch (SURVEY.md
    8(d): 2 n m d flops; bytes 4 d (n + m) + 12 n k) over its launch time."""
    n, d, k = cfg["n"], cfg["d"], cfg["k"]
    t = per_launch_ms / 1e3
    out = {"kernel": name, "per_launch_ms": round(per_launch_ms, 4), "launches": launches}
    if name.startswith("merge"):
        alg = n * world * k * 12 + n * k * 12
        out.update(bound="hbm", unit="GB/s", peak=peaks["hbm_gbs"], achieved=alg / t / 1e9,
                   work=f"{alg} algorithmic bytes per launch (gathered lists in, table out)")
    elif "filter" in name:
        alg = 2.0 * n * m_local * d
        out.update(bound="tensor", unit="TFLOP/s", peak=peaks["bf16_tflops"],
                   achieved=alg / t / 1e12,
                   work=f"2 n m d = {alg:.4g} flops per launch (n={n}, m={m_local}, d={d})")
    elif "exact" in name:  # the FP32 SIMT path (L1 / Linf, d > 128, certificate fallback)
        alg = 2.0 * n * m_local * d
        out.update(bound="fp32", unit="TFLOP/s", peak=FP32_SIMT_TFLOPS,
                   achieved=alg / t / 1e12,
                   work=f"2 n m d = {alg:.4g} flops per launch on the FP32 pipe")

    else:
        alg = 4.0 * d * (n + m_local) + 12.0 * n * k
        out.update(bound="hbm", unit="GB/s", peak=peaks["hbm_gbs"], achieved=alg / t / 1e9,
                   work=f"4 d (n + m) + 12 n k = {alg:.4g} algorithmic bytes per launch")
    out["frac"] = round(out["achieved"] / out["peak"], 4)
    out["achieved"] = round(out["achieved"], 3)
    if out["bound"] == "fp32":
        out["peak_source"] = ("nominal FP32 SIMT peak, 148 SMs x 128 lanes x 2 flops x 1.965 GHz "
                              "(MEASURED_PEAKS.json has no FP32 figure)")
    else:
        src = "bf16 dense" if out["bound"] == "tensor" else "hbm"
        out["peak_source"] = f"{peak_src} (MEASURED_PEAKS.json {src})"
    # the committed ncu capture is of config B (m = n = 38400, d = 96, k = 20):
    # its DRAM bytes describe that shape only
    shape_b = (cfg.get("m"), cfg.get("n"), cfg.get("d"), cfg.get("k")) == (38400, 38400, 96, 20)
    out["traffic"] = measured_traffic(name) if shape_b and world == 1 else None
    return out


def regime_metrics(cfg, m_local, step_ms, alg_bytes):
    """Low-d / large-k regime: selection-bound, so report the
    achieved HBM rate of the algorithmic bytes and candidate visits/s (n m / t)
    against the SM thread-instruction issue capacity."""
    t = step_ms / 1e3
    visits = cfg["n"] * m_local / t
    return {"regime": "selection-bound" if cfg["d"] <= 32 or cfg["k"] >= 100 else "compute-bound",
            "candidate_visits_per_s": round(visits, 1),
            "issue_capacity_thread_inst_per_s": ISSUE_THREAD_INST_PER_S,
            "visits_per_issue_slot": round(visits / ISSUE_THREAD_INST_PER_S, 4),
            "hbm_gbs_of_algorithmic_bytes": round(alg_bytes / t / 1e9, 2)}


def run_line(be, plumb, letter, cfg, args, world, rank, path):
    """One JSON line: warm-up, two profiled untimed steps, K timed steps, e2e,
    correctness gate, CPU baseline.  Runs on every rank; rank 0 prints."""
    n, m, d, k = cfg["n"], cfg["m"], cfg["d"], cfg["k"]
    from paper_0804_1448_b200.sharding import check_shardable
    check_shardable(m, world, k)
    lo, hi = shard_bounds(m, world, rank)
    m_local = hi - lo
    sr, sq = seeds(cfg)
    # synthetic inputs on the device: rows lo..hi of R (counter stream offset),
    # all of Q -- the same values the oracle's host generator produces
    R = be.empty((m_local, d))
    Q = be.empty((n, d))
    be.fill_uniform(R, sr, lo * d)
    be.fill_uniform(Q, sq, 0)
    be.sync()
    index = be.index(R, m_local, d, lo)
    od = be.empty((n, k))
    oi = be.empty((n, k), "i64")
    comm = None
    if world > 1:
        uid = plumb.broadcast_bytes(be.unique_id() if rank == 0 else None)
        comm = be.comm(uid, world, rank)
    elif os.environ.get("KNN_BENCH_FORCE_DIST"):  # dev: the N > 1 step on a 1-rank communicator
        comm = be.comm(be.unique_id(), 1, 0)

    def step():
        if comm is None:
            be.search(index, Q, n, k, od, oi, path)
        else:
            be.dist_search(comm, index, Q, n, k, od, oi, path)

    clocks = be.clocks()
    clocks.start()
    for _ in range(args.warmup):
        step()
    be.sync()
    # per-kernel breakdown from two untimed, fully profiled steps (events around
    # every launch perturb the step); it names the dominant kernel, which alone
    # is bracketed by events inside the timed region
    be.profile_enable(True)
    for _ in range(2):
        be.flush_l2()
        step()
    be.sync()
    be.profile_enable(False)
    breakdown = be.profile_collect()
    cand = [kk for kk in breakdown if not kk.startswith("fill")]
    dom_name = max(cand, key=lambda kk: breakdown[kk][0]) if cand else ""
    starts = [be.event() for _ in range(args.steps)]
    ends = [be.event() for _ in range(args.steps)]
    if plumb:
        plumb.barrier()
    be.sync()
    be.reset_launch_count()
    be.profile_enable(True, only=dom_name)
    t_lo = time.perf_counter()
    for i in range(args.steps):
        be.flush_l2()
        be.record(starts[i])
        step()
        be.record(ends[i])
    be.sync()
    t_hi = time.perf_counter()
    if plumb:
        plumb.barrier()
    be.profile_enable(False)
    launches = be.launch_count()
    prof = be.profile_collect()
    be.profile_enable(False, only="")
    clocks.window = (t_lo, t_hi)
    clocks.stop()
    total_ms = sum(be.elapsed_ms(s, e) for s, e in zip(starts, ends))
    if plumb:
        total_ms = plumb.max(total_ms)
    ms_per_step = total_ms / args.steps
    value = n / (ms_per_step / 1e3)

    peaks, peak_src = load_peaks()
    dom_ms, dom_cnt = prof.get(dom_name, (0.0, 0))
    per_launch_ms = dom_ms / max(dom_cnt, 1)
    if plumb:
        per_launch_ms = plumb.max(per_launch_ms)
    roofline = dominant_roofline(dom_name, per_launch_ms, dom_cnt, cfg, m_local, world, peaks,
                                 peak_src)
    roofline["timing"] = "the dominant kernel bracketed by CUDA events inside the timed region"
    roofline["kernels"] = {kk: {"ms_per_launch": round(v[0] / max(v[1], 1), 4), "launches": v[1]}
                           for kk, v in breakdown.items()}
    roofline["kernels_source"] = "2 untimed profiled steps (events around every launch)"
    if world > 1:
        roofline["per_gpu"] = f"rank-local shard of m={m_local}; max over ranks"
    alg_bytes = 4.0 * d * (n + m_local) + 12.0 * n * k
    if d <= 32 or k >= 100:
        roofline["selection_regime"] = regime_metrics(cfg, m_local, ms_per_step, alg_bytes)

    # the same search as one bf_knn call on device buffers: the reference set
    # is prepared inside the timed call (range, scale, fp16 convert of R)
    oneshot = None
    if world == 1 and hasattr(be, "search_oneshot"):
        be.search_oneshot(R, m_local, Q, n, d, k, od, oi, path)
        be.sync()
        s1 = [be.event() for _ in range(args.steps)]
        e1 = [be.event() for _ in range(args.steps)]
        for i in range(args.steps):
            be.flush_l2()
            be.record(s1[i])
            be.search_oneshot(R, m_local, Q, n, d, k, od, oi, path)
            be.record(e1[i])
        be.sync()
        ms1 = sum(be.elapsed_ms(a, b) for a, b in zip(s1, e1)) / args.steps
        oneshot = {"value": round(n / (ms1 / 1e3), 2), "unit": "queries/s", "ms_per_step": round(ms1, 5),
                   "api": "knn_b200_search_device (device buffers, reference set prepared in the call)",
                   "timing": "CUDA events on the launch stream, L2 flushed between steps"}
    e2e = run_e2e(be, plumb, args, world, rank, cfg, lo, hi, path, sr, sq)
    oi_h = be.host(oi)
    od_h = be.host(od)
    gate = correctness_gate(cfg, oi_h, od_h, sr, sq) if rank == 0 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, sr, sq, target_s=args.cpu_seconds)
    if comm is not None:
        comm.close()
    index.close()
    # N > 1: the same workload on this one GPU (all of R), so the line carries
    # its own single-GPU baseline for the scaling ratio (BENCH's N = 1 line is
    # the config-B headline, a different workload)
    single = None
    if (world > 1 or os.environ.get("KNN_BENCH_FORCE_SINGLE")) and rank == 0:  # env: dev check on 1 GPU
        Rf = be.empty((m, d))
        be.fill_uniform(Rf, sr, 0)
        ixf = be.index(Rf, m, d, 0)
        be.search(ixf, Q, n, k, od, oi, path)
        be.sync()
        reps = max(2, min(args.steps, 5))
        s2 = [be.event() for _ in range(reps)]
        e2 = [be.event() for _ in range(reps)]
        for i in range(reps):
            be.flush_l2()
            be.record(s2[i])
            be.search(ixf, Q, n, k, od, oi, path)
            be.record(e2[i])
        be.sync()
        ms2 = sum(be.elapsed_ms(a, b) for a, b in zip(s2, e2)) / reps
        ixf.close()
        del Rf
        single = {"n_gpus": 1, "value": round(n / (ms2 / 1e3), 1), "unit": "queries/s",
                  "ms_per_step": round(ms2, 5), "steps": reps,
                  "ratio": round(value / (n / (ms2 / 1e3)), 3),
                  "note": "rank 0 alone, all of R on its GPU, same index search; "
                          "ratio = this line's value / this value"}
    if rank != 0:
        return None
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": round(value / PAPER_B_QPS, 2) if letter == "B" else None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(letter, cfg), "m": m, "n": n, "d": d, "k": k,
                   "metric": "euclidean",
                   "parallelism": "single" if world == 1 else f"reference-sharded x{world} "
                                  "(NCCL all-gather + device merge)",
                   "path": args.path,
                   "l2": "flushed between timed steps (256 MiB write, then a 256 MiB read "
                         "that evicts the dirty lines)",
                   "inputs": "uniform [0,1) fp32, splitmix64 counter stream, seeds "
                             "derive_seed(42,m,d,0)/(42,n,d,1); R rows of each shard at their "
                             "global counter offset",
                   "vs_baseline_ref": "paper Table 1 BF-CUDA 8800 GTX, 878 q/s" if letter == "B"
                   else "no published number for this config"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "device_one_shot": oneshot,
        "single_gpu_same_workload": single,
        "gpu_launches": launches,
        "correctness_gate": gate, "clocks": clocks.summary(),
    }


def run_rho_line(be, letter, cfg, args):
    """--task rho_k: the entropy estimator's self-join (entropy.cpp:75-89,
    rho_k_all) on the config's reference set: one device search of every
    point against the set with k + 1, self excluded by index in the epilogue.
    value = points/s."""
    torch, knn = be.torch, be.knn
    m, d, k = cfg["m"], cfg["d"], cfg["k"]
    sr, _ = seeds(cfg)
    P = be.empty((m, d))
    be.fill_uniform(P, sr, 0)
    out = torch.empty(m, dtype=torch.float64, device=be.dev)
    step = lambda: knn.rho_k_all_device(P.data_ptr(), m, d, k, out.data_ptr(), stream=be.sptr)
    for _ in range(args.warmup):
        step()
    be.sync()
    ev = [(be.event(), be.event()) for _ in range(args.steps)]
    be.reset_launch_count()
    for a, b in ev:
        be.flush_l2()
        be.record(a)
        step()
        be.record(b)
    be.sync()
    launches = be.launch_count()
    ms = sum(be.elapsed_ms(a, b) for a, b in ev) / args.steps
    got = out.cpu().numpy()
    from oracle.oracle import Oracle, Reference
    orc = Oracle()
    Ph = orc.counter_f32(m, d, sr)
    pick = np.linspace(0, m - 1, 256).astype(np.int64)
    ri, rd = orc.knn(Ph[pick], Ph, k + 1)
    want = np.array([[x for j, x in zip(ri[t], rd[t]) if j != pick[t]][k - 1]
                     for t in range(len(pick))])
    ok = bool(np.allclose(got[pick], want, rtol=1e-5, atol=0))
    if not ok:
        print(json.dumps({"error": "rho_k correctness gate failed"}), file=sys.stderr)
        sys.exit(1)
    cpu = None
    if not args.no_cpu_baseline:
        ref = Reference()
        s = 2000
        t0 = time.perf_counter()
        ref.bf_knn(Ph[:s].astype(np.float64), Ph.astype(np.float64), k + 1)
        t = time.perf_counter() - t0
        cpu = {"value": round(s / t, 2), "unit": "points/s", "cores": ref.max_threads(),
               "kind": "reference", "sample": f"knn::bf_knn(first {s} points, all {m}, k+1={k + 1}), "
               "the search inside knn::rho_k_all (entropy.cpp:84)"}
    return {"metric": "rho_k_all points/sec (self-join, entropy.cpp:75-89)",
            "value": round(m / (ms / 1e3), 1), "unit": "points/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"rho_k_all over {workload_name(letter, cfg)} points",
                       "n": m, "d": d, "k": k, "task": "rho_k"},
            "gpu_launches": launches, "cpu_baseline": cpu,
            "correctness_gate": {"points_checked": 256, "result": "pass",
                                 "oracle": "oracle/knn_oracle.c k+1 search, self dropped by index"}}


def correctness_gate(cfg, oi, od, sr, sq, sample: int = 256):
    """Checker only (never timed): the oracle's top-k of a query sample spread
    over the whole query set (same counter-stream inputs, generated on the
    host) vs the table the timed steps left in HBM.  Exits without printing a
    result line on failure."""
    from oracle.oracle import Oracle, compare
    n, m, d, k = cfg["n"], cfg["m"], cfg["d"], cfg["k"]
    orc = Oracle()
    if m * n * d > 2e13:  # config E: keep the host check to seconds
        sample = 48
    pick = np.linspace(0, n - 1, min(sample, n)).astype(np.int64)
    Rh = orc.counter_f32(m, d, sr)
    Qh = orc.counter_f32(n, d, sq)[pick]
    ri, rd = orc.knn(Qh, Rh, k)
    rep = compare(oi[pick], od[pick], ri, rd, Qh, Rh, oracle=orc)
    if not rep.ok:
        print(json.dumps({"error": "correctness gate failed", "config": cfg, "report": str(rep)}),
              file=sys.stderr, flush=True)
        sys.exit(1)
    return {"queries_checked": int(len(pick)),
            "oracle": "oracle/knn_oracle.c (pinned to the reference's bf_knn)",
            "comparator": "distance rel 1e-5, index only at near-ties", "result": "pass",
            "max_rel_err": float(rep.max_rel), "near_tie_index_swaps": int(rep.near_tie_mismatches)}


def run_e2e(be, plumb, args, world, rank, cfg, lo, hi, path, sr, sq):
    """Same metric end to end: host buffers in, host table out, copies timed."""
    n, m, d, k = cfg["n"], cfg["m"], cfg["d"], cfg["k"]
    if not hasattr(be, "torch"):
        return None
    torch, knn = be.torch, be.knn
    from oracle.oracle import Oracle  # the host copy of the same synthetic inputs
    orc = Oracle()
    Qh = torch.from_numpy(orc.counter_f32(n, d, sq)).pin_memory()
    Rh = torch.from_numpy(orc.counter_f32(hi - lo, d, sr, row_begin=lo)).pin_memory()
    od = torch.empty((n, k), dtype=torch.float32).pin_memory()
    oi = torch.empty((n, k), dtype=torch.int64).pin_memory()
    qn, rn, odn, oin = Qh.numpy(), Rh.numpy(), od.numpy(), oi.numpy()
    if world == 1:
        conf = knn.BfConfig(path=path)

        def step():
            knn.bf_knn(qn, rn, k, config=conf, out=(odn, oin))
        h2d = (n + m) * d * 4
        d2h = n * k * (4 + 8)
        api = "knn_b200_search (bf_knn drop-in; pinned host buffers)"
    else:
        dq = be.empty((n, d))
        dr = be.empty((hi - lo, d))
        fd = be.empty((n, k))
        fi = be.empty((n, k), "i64")
        uid = plumb.broadcast_bytes(be.unique_id() if rank == 0 else None)
        comm = be.comm(uid, world, rank)

        def step():
            dq.copy_(Qh, non_blocking=True)
            dr.copy_(Rh, non_blocking=True)
            be.sync()
            ix = be.index(dr, hi - lo, d, lo)
            be.dist_search(comm, ix, dq, n, k, fd, fi, path)
            if rank == 0:
                od.copy_(fd, non_blocking=True)
                oi.copy_(fi, non_blocking=True)
            be.sync()
            ix.close()
        h2d = (n + (hi - lo)) * d * 4
        d2h = n * k * 12 if rank == 0 else 0
        api = ("per rank: H2D of its reference shard and the queries, knn_b200_index_create_device "
               "(prep), knn_b200_dist_search_device (NCCL all-gather + merge), D2H on rank 0")
    for _ in range(max(1, min(args.warmup, 3))):
        step()
    be.sync()
    if plumb:
        plumb.barrier()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    if plumb:
        tot = plumb.max(tot)
    if world > 1:
        comm.close()
    return {"value": round(n / (tot / args.steps), 1), "unit": "queries/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(tot / args.steps * 1e3, 4), "api": api,
            "timing": "wall clock per step (host buffers), max over ranks"}


# ---------------------------------------------------------- CPU baselines ----
def _ref():
    from oracle.oracle import Reference
    return Reference()


def _host_inputs(cfg, sr, sq, nq):
    from oracle.oracle import Oracle
    orc = Oracle()
    R = orc.counter_f32(cfg["m"], cfg["d"], sr).astype(np.float64)
    Q = orc.counter_f32(nq, cfg["d"], sq).astype(np.float64)
    return Q, R


def cpu_baseline(cfg, sr, sq, target_s: float = 10.0):
    """The reference's own bf_knn on the host cores, bounded query sample."""
    ref = _ref()
    k = cfg["k"]
    big = cfg["m"] * cfg["d"] > 2e8
    chunk = 64 if big else 1024  # 1024 x m doubles would be 82 GB at config E
    Q, R = _host_inputs(cfg, sr, sq, min(cfg["n"], 4096))
    ref.bf_knn(Q[:4], R, k, chunk=chunk)  # warm-up (thread spin-up, first touch)
    probe = 8 if big else 64
    t0 = time.perf_counter()
    ref.bf_knn(Q[:probe], R, k, chunk=chunk)
    tp = time.perf_counter() - t0
    s = int(min(Q.shape[0], max(probe, probe * target_s / max(tp, 1e-6))))
    t0 = time.perf_counter()
    ref.bf_knn(Q[:s], R, k, chunk=chunk)
    t = time.perf_counter() - t0
    return {"value": round(s / t, 2), "unit": "queries/s", "cores": ref.max_threads(),
            "kind": "reference",
            "sample": f"first {s} of {cfg['n']} queries vs the full m={cfg['m']} reference set "
                      f"(d={cfg['d']}, k={k}); knn::bf_knn from oracle/_ref/libknnref.so, "
                      f"BfConfig chunk_size={chunk}, all OpenMP threads",
            "seconds": round(t, 3)}


def run_reference(args, letter):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    try:
        ref = _ref()
    except FileNotFoundError as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return
    for cfg in CONFIGS[letter][1]:
        n, m, d, k = cfg["n"], cfg["m"], cfg["d"], cfg["k"]
        sr, sq = seeds(cfg)
        big = m * d > 2e8
        chunk = 64 if big else 1024
        Q, R = _host_inputs(cfg, sr, sq, min(n, 8192))
        ref.bf_knn(Q[:4], R, k, chunk=chunk)
        probe = 4 if big else 64
        t0 = time.perf_counter()
        ref.bf_knn(Q[:probe], R, k, chunk=chunk)
        tp = time.perf_counter() - t0
        per_step = min(10.0, 150.0 / max(1, args.steps + args.warmup))
        s = int(min(Q.shape[0], max(4 if big else 32, probe * per_step / max(tp, 1e-6))))
        for _ in range(args.warmup):
            ref.bf_knn(Q[:s], R, k, chunk=chunk)
        times = []
        for i in range(args.steps):
            q0 = (i * s) % max(1, Q.shape[0] - s)
            t0 = time.perf_counter()
            ref.bf_knn(Q[q0:q0 + s], R, k, chunk=chunk)
            times.append(time.perf_counter() - t0)
        ms = statistics.mean(times) * 1e3
        value = s / (ms / 1e3)
        sample = (f"{s} of {n} queries per step vs the full m={m} reference set (d={d}, k={k}); "
                  "knn::bf_knn from oracle/_ref/libknnref.so (reference sources, -O3 -fopenmp "
                  f"-ffp-contract=off), BfConfig chunk_size={chunk}")
        line = {"metric": METRIC, "value": round(value, 2), "unit": "queries/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": workload_name(letter, cfg), "m": m, "n": n, "d": d, "k": k,
                           "metric": "euclidean", "parallelism": "host OpenMP"},
                "cpu_baseline": {"value": round(value, 2), "unit": "queries/s",
                                 "cores": ref.max_threads(), "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": round(value, 2), "unit": "queries/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ launcher --
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args):
    """--gpus N > 1 without torchrun: start N ranks (one per GPU) ourselves;
    never fall back to a 1-GPU run."""
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:
        have = 0
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but {have} GPU(s) visible",
                          "n_gpus": args.gpus}), flush=True)
        return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_ours(args, letter):
    world, rank, local = dist_env()
    if world != args.gpus and args.gpus != 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    be = CudaBackend(local)
    plumb = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=be.dev)
        plumb = DistPlumbing(world, rank, "nccl")
    path = {"auto": 0, "exact": 1, "tensor": 2}[args.path]
    if args.task == "rho_k":
        for cfg in CONFIGS[letter][1]:
            print(json.dumps(run_rho_line(be, letter, cfg, args)), flush=True)
        return
    for cfg in CONFIGS[letter][1]:
        line = run_line(be, plumb, letter, cfg, args, world, rank, path)
        if line is not None:
            print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=None,
                    help="BASELINE.json config (default: B on 1 GPU, E on N > 1)")
    ap.add_argument("--path", choices=["auto", "exact", "tensor"], default="auto")
    ap.add_argument("--task", choices=["search", "rho_k"], default="search",
                    help="rho_k: the entropy self-join (rho_k_all) on the config's points")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    return args


def main():
    args = parse()
    world, _, _ = dist_env()
    letter = args.config or ("B" if max(world, args.gpus) == 1 else "E")
    if args.impl == "reference":
        run_reference(args, letter)
        return 0
    if args.gpus > 1 and world == 1:
        return self_launch(args)
    run_ours(args, letter)
    return 0


if __name__ == "__main__":
    sys.exit(main())
