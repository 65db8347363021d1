#!/usr/bin/env python3
"""Benchmark: kNN queries/s on BASELINE.json configs[1] (m=n=38400, d=96, k=20).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

ours (default)
    A "step" is one full search of all n queries against the reference set,
    inputs already resident in HBM.  N=1: one device search.  N>1 (launched by
    torchrun, one rank per GPU): the reference set is sharded into contiguous
    index ranges, every rank searches its shard (raw keys, global indices),
    the per-shard top-k lists are all-gathered over NCCL and merged on device
    (SURVEY.md 8(e)); total work is fixed, so scaling is "strong".
    Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA
    events on the launch stream with an L2 flush (256 MiB write, then a
    256 MiB read that evicts the dirty lines) between
    steps; barrier + synchronize around the timed region; max over ranks.
    e2e: the same metric through the public host API (pinned host Q/R in,
    host results out, H2D/D2H inside the timed region).
    roofline: the dominant kernel's per-launch time from CUDA events recorded
    around each of its launches on its stream inside the timed region (engine
    profiling hooks, restricted to that kernel so the other launches run
    unperturbed), against MEASURED_PEAKS.json; the per-kernel breakdown comes
    from two untimed, fully profiled steps.
    cpu_baseline (rank 0, N=1): the reference's own bf_knn (oracle/_ref),
    all host threads, on a bounded query sample of the same inputs.

reference (--impl reference)
    Rank 0 only: the reference's CPU bf_knn on the box's host cores, each step
    a bounded query sample of the same workload; other ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_B = dict(m=38400, n=38400, d=96, k=20)
PAPER_B_QPS = 38400 / 43.74  # BF-CUDA 43.74 s on a GeForce 8800 GTX
METRIC = "kNN queries/sec (m=n=38400, d=96, k=20) at 1/2/4/8 B200 vs CPU ref"


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


# ------------------------------------------------------------------ our arm --
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_0804_1448_b200 as knn

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = dict(CONFIG_B)
    n, m, d, k = cfg["n"], cfg["m"], cfg["d"], cfg["k"]
    path = {"auto": knn.PATH_AUTO, "exact": knn.PATH_EXACT, "tensor": knn.PATH_TENSOR}[args.path]
    # a dedicated (non-default) stream: the engine, the L2 flush, the step
    # events and NCCL all order on it (handle 0 would mean "engine stream")
    torch.cuda.set_stream(torch.cuda.Stream(dev))
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    assert sptr != 0

    # synthetic inputs, generated on the device (counter-based splitmix64)
    sr, sq = seeds(cfg)
    R = torch.empty((m, d), dtype=torch.float32, device=dev)
    Q = torch.empty((n, d), dtype=torch.float32, device=dev)
    knn.fill_uniform_device(R.data_ptr(), m * d, sr, 0, sptr)
    knn.fill_uniform_device(Q.data_ptr(), n * d, sq, 0, sptr)
    from paper_0804_1448_b200.sharding import check_shardable, shard_bounds
    check_shardable(m, world, k)
    lo, hi = shard_bounds(m, world, rank)
    Rs = R[lo:hi]
    index = knn.Index(device_ptr=Rs.data_ptr(), m=hi - lo, d=d, index_base=lo, device=local)
    out_d = torch.empty((n, k), dtype=torch.float32, device=dev)
    out_i = torch.empty((n, k), dtype=torch.int64, device=dev)
    if world > 1:
        loc_k = torch.empty((n, k), dtype=torch.float32, device=dev)
        loc_i = torch.empty((n, k), dtype=torch.int64, device=dev)
        all_k = torch.empty((world, n, k), dtype=torch.float32, device=dev)
        all_i = torch.empty((world, n, k), dtype=torch.int64, device=dev)

    def step():
        if world == 1:
            index.search_device(Q.data_ptr(), n, k, out_d.data_ptr(), out_i.data_ptr(),
                                path=path, stream=sptr)
        else:
            index.search_device(Q.data_ptr(), n, k, loc_k.data_ptr(), loc_i.data_ptr(),
                                path=path, stream=sptr, raw_keys=True)
            dist.all_gather_into_tensor(all_k, loc_k)
            dist.all_gather_into_tensor(all_i, loc_i)
            knn.merge_device(all_k.data_ptr(), all_i.data_ptr(), world, n, k, out_d.data_ptr(),
                             out_i.data_ptr(), stream=sptr)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # a second buffer read after the flush write evicts the flush's dirty lines,
    # so their write-back lands before the step's start event, not inside it
    clean = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, L2 flushed between them (outside the events)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    # per-kernel breakdown from two untimed, fully profiled steps (events around
    # every launch perturb the step by ~30 us); it names the dominant kernel,
    # which alone is bracketed by events inside the timed region
    knn.profile_enable(True)
    for _ in range(2):
        flush.zero_()
        clean.sum()
        step()
    torch.cuda.synchronize(dev)
    knn.profile_enable(False)
    breakdown = knn.profile_collect()
    dom_name = max((kk for kk in breakdown if not kk.startswith("fill")),
                   key=lambda kk: breakdown[kk][0])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    knn.reset_launch_count()
    knn.profile_enable(True, only=dom_name)
    t_lo = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        clean.sum()
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize(dev)
    t_hi = time.perf_counter()
    if world > 1:
        dist.barrier()
    knn.profile_enable(False)
    launches = knn.launch_count()
    prof = knn.profile_collect()
    knn.profile_enable(False, only="")
    clocks.window = (t_lo, t_hi)
    clocks.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = n / (ms_per_step / 1e3)

    # ---- dominant kernel roofline (per-launch, events on its launch stream)
    peaks, peak_src = load_peaks()
    flush_ms = 0.0
    dom_ms, dom_cnt = prof.get(dom_name, (0.0, 0))
    per_launch_ms = dom_ms / max(dom_cnt, 1)
    m_local = hi - lo
    if dom_name.startswith("merge"):
        alg = n * world * k * 12 + n * k * 12
        bound, unit, peak = "hbm", "GB/s", peaks["hbm_gbs"]
        achieved = alg / (per_launch_ms / 1e3) / 1e9
    else:
        # algorithmic work of one search launch: 2*n*m_local*d flops
        alg = 2.0 * n * m_local * d
        bound, unit = "tensor", "TFLOP/s"
        peak = peaks["bf16_tflops"]
        achieved = alg / (per_launch_ms / 1e3) / 1e12
    roofline = {"bound": bound, "achieved": round(achieved, 3), "peak": peak, "unit": unit,
                "frac": round(achieved / peak, 4), "traffic": measured_traffic(dom_name),
                "kernel": dom_name, "per_launch_ms": round(per_launch_ms, 4),
                "launches": dom_cnt, "peak_source": f"{peak_src} (MEASURED_PEAKS.json bf16 dense)"
                if bound == "tensor" else f"{peak_src} (MEASURED_PEAKS.json hbm)",
                "timing": "the dominant kernel bracketed by CUDA events inside the timed region",
                "kernels": {kk: {"ms_per_launch": round(v[0] / max(v[1], 1), 4), "launches": v[1]}
                            for kk, v in breakdown.items()},
                "kernels_source": "2 untimed profiled steps (events around every launch)"}

    # ---- e2e through the public host API (pinned host buffers)
    e2e = run_e2e(args, knn, torch, dist, dev, world, rank, Q, R, lo, hi, cfg, path)

    # ---- correctness gate (bench.cpp:148-157): the table the
    # timed steps produced, on a query sample spread over all query tiles, must
    # pass the north-star comparator against the oracle before a number is printed
    oi = out_i.cpu().numpy()
    od = out_d.cpu().numpy()
    gate = correctness_gate(Q, R, oi, od, k) if rank == 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(Q, R, cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": round(value / PAPER_B_QPS, 2), "dtype": "f32", "data": "synthetic",
            "config": {"workload": "configs[1]: m=n=38400, d=96, k=20, euclidean",
                       "m": m, "n": n, "d": d, "k": k, "metric": "euclidean",
                       "parallelism": "single" if world == 1 else f"reference-sharded x{world}",
                       "path": args.path, "l2": "flushed between timed steps (256 MiB write, then a 256 MiB read that evicts the dirty lines)",
                       "inputs": "uniform [0,1) fp32, splitmix64 counter stream, "
                                 "seeds derive_seed(42,m,d,0)/(42,n,d,1)",
                       "vs_baseline_ref": "paper Table 1 BF-CUDA 8800 GTX, 878 q/s"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "correctness_gate": gate,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    index.close()
    if world > 1:
        dist.destroy_process_group()


def correctness_gate(Q, R, oi, od, k, sample: int = 256):
    """Checker only (never timed): oracle top-k of `sample` queries spread over
    the whole query set vs the table the timed steps left in HBM.  Exits
    without printing a result line on failure."""
    from oracle.oracle import Oracle, compare
    n = oi.shape[0]
    pick = np.linspace(0, n - 1, min(sample, n)).astype(np.int64)
    Qh = Q.cpu().numpy()[pick]
    Rh = R.cpu().numpy()
    orc = Oracle()
    ri, rd = orc.knn(Qh, Rh, k)
    rep = compare(oi[pick], od[pick], ri, rd, Qh, Rh, oracle=orc)
    if not rep.ok:
        print(json.dumps({"error": "correctness gate failed", "report": str(rep)}),
              file=sys.stderr, flush=True)
        sys.exit(1)
    return {"queries_checked": int(len(pick)), "oracle": "oracle/knn_oracle.c (pinned to the "
            "reference's bf_knn)", "comparator": "distance rel 1e-5, index only at near-ties",
            "result": "pass", "max_rel_err": float(getattr(rep, "max_rel", 0.0))}


def run_e2e(args, knn, torch, dist, dev, world, rank, Q, R, lo, hi, cfg, path):
    n, m, d, k = cfg["n"], cfg["m"], cfg["d"], cfg["k"]
    Qh = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    Rh = torch.empty((hi - lo, d), dtype=torch.float32, pin_memory=True)
    Qh.copy_(Q.cpu())
    Rh.copy_(R[lo:hi].cpu())
    od = torch.empty((n, k), dtype=torch.float32, pin_memory=True)
    oi = torch.empty((n, k), dtype=torch.int64, pin_memory=True)
    qn, rn, odn, oin = Qh.numpy(), Rh.numpy(), od.numpy(), oi.numpy()
    conf = knn.BfConfig(path=path)
    if world == 1:
        def step():
            knn.bf_knn(qn, rn, k, config=conf, out=(odn, oin))
        h2d = (n + m) * d * 4
        d2h = n * k * (4 + 8)
    else:
        dq = torch.empty((n, d), dtype=torch.float32, device=dev)
        dr = torch.empty((hi - lo, d), dtype=torch.float32, device=dev)
        lk = torch.empty((n, k), dtype=torch.float32, device=dev)
        li = torch.empty((n, k), dtype=torch.int64, device=dev)
        ak = torch.empty((world, n, k), dtype=torch.float32, device=dev)
        ai = torch.empty((world, n, k), dtype=torch.int64, device=dev)
        fd = torch.empty((n, k), dtype=torch.float32, device=dev)
        fi = torch.empty((n, k), dtype=torch.int64, device=dev)
        sptr = torch.cuda.current_stream(dev).cuda_stream

        def step():
            dq.copy_(Qh, non_blocking=True)
            dr.copy_(Rh, non_blocking=True)
            knn.search_device(dq.data_ptr(), n, dr.data_ptr(), hi - lo, d, k, lk.data_ptr(),
                              li.data_ptr(), path=path, stream=sptr, raw_keys=True)
            li.add_(lo)
            dist.all_gather_into_tensor(ak, lk)
            dist.all_gather_into_tensor(ai, li)
            knn.merge_device(ak.data_ptr(), ai.data_ptr(), world, n, k, fd.data_ptr(),
                             fi.data_ptr(), stream=sptr)
            if rank == 0:
                od.copy_(fd, non_blocking=True)
                oi.copy_(fi, non_blocking=True)
            torch.cuda.synchronize(dev)
        h2d = (n + (hi - lo)) * d * 4
        d2h = n * k * 12 if rank == 0 else 0
    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    if world > 1:
        t = torch.tensor([tot], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = float(t.item())
    return {"value": round(n / (tot / args.steps), 1), "unit": "queries/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(tot / args.steps * 1e3, 4),
            "api": "knn_b200_search (host buffers, pinned)" if world == 1 else
                   "H2D + knn_b200_search_device + NCCL all_gather + knn_b200_merge_device + D2H"}


# ---------------------------------------------------------- CPU baselines ----
def _ref():
    from oracle.oracle import Reference
    return Reference()


def cpu_baseline(Q, R, cfg, target_s: float = 10.0):
    """The reference's own bf_knn on the host cores, bounded query sample."""
    ref = _ref()
    Rh = R.cpu().numpy().astype(np.float64)
    Qh = Q.cpu().numpy().astype(np.float64)
    k = cfg["k"]
    ref.bf_knn(Qh[:16], Rh, k)  # warm-up (thread spin-up, first touch)
    t0 = time.perf_counter()
    ref.bf_knn(Qh[:64], Rh, k)
    t64 = time.perf_counter() - t0
    s = int(min(Qh.shape[0], max(64, 64 * target_s / max(t64, 1e-6))))
    t0 = time.perf_counter()
    ref.bf_knn(Qh[:s], Rh, k)
    t = time.perf_counter() - t0
    return {"value": round(s / t, 2), "unit": "queries/s", "cores": ref.max_threads(),
            "kind": "reference",
            "sample": f"first {s} of {Qh.shape[0]} queries vs the full m={Rh.shape[0]} "
                      f"reference set (d={Rh.shape[1]}, k={k}); knn::bf_knn from "
                      "oracle/_ref/libknnref.so, default BfConfig (all OpenMP threads)",
            "seconds": round(t, 3)}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Oracle
    try:
        ref = _ref()
    except FileNotFoundError as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return
    orc = Oracle()
    cfg = dict(CONFIG_B)
    n, m, d, k = cfg["n"], cfg["m"], cfg["d"], cfg["k"]
    sr, sq = seeds(cfg)
    R = orc.counter_f32(m, d, sr).astype(np.float64)
    Q = orc.counter_f32(n, d, sq).astype(np.float64)
    ref.bf_knn(Q[:16], R, k)
    t0 = time.perf_counter()
    ref.bf_knn(Q[:64], R, k)
    t64 = time.perf_counter() - t0
    per_step = min(10.0, 150.0 / max(1, args.steps + args.warmup))
    s = int(min(n, max(32, 64 * per_step / max(t64, 1e-6))))
    for i in range(args.warmup):
        ref.bf_knn(Q[:s], R, k)
    times = []
    for i in range(args.steps):
        lo = (i * s) % max(1, n - s)
        t0 = time.perf_counter()
        ref.bf_knn(Q[lo:lo + s], R, k)
        times.append(time.perf_counter() - t0)
    ms = statistics.mean(times) * 1e3
    value = s / (ms / 1e3)
    sample = (f"{s} of {n} queries per step vs the full m={m} reference set (d={d}, k={k}); "
              "knn::bf_knn from oracle/_ref/libknnref.so (reference sources, -O3 -fopenmp "
              "-ffp-contract=off), default BfConfig")
    line = {"metric": METRIC, "value": round(value, 2), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "configs[1]: m=n=38400, d=96, k=20, euclidean", "m": m,
                       "n": n, "d": d, "k": k, "parallelism": "host OpenMP"},
            "cpu_baseline": {"value": round(value, 2), "unit": "queries/s",
                             "cores": ref.max_threads(), "kind": "reference", "sample": sample},
            "e2e": {"value": round(value, 2), "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--path", choices=["auto", "exact", "tensor"], default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
