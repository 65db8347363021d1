"""ctypes loaders for the parity oracles -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
reference arm may import this module.  The product package never does.

Two oracles:

* ``Oracle`` -- ``oracle/lib/liboracle.so``, the plain-C restatement in
  ``knn_oracle.c`` (always buildable with gcc).
* ``Reference`` -- ``oracle/_ref/libknnref.so``, the reference's own
  ``knn::bf_knn`` / ``knn::reference_knn`` compiled from
  ``/root/reference/proj/src`` (see ``oracle/Makefile``), wrapped by
  ``ref_capi.cpp``.

Also the north-star tolerance comparator.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libknnref.so")

EUCLIDEAN, MANHATTAN, CHEBYSHEV, MAHALANOBIS = 0, 1, 2, 3
METRICS = {"euclidean": EUCLIDEAN, "manhattan": MANHATTAN, "chebyshev": CHEBYSHEV,
           "mahalanobis": MAHALANOBIS}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


class Oracle:
    """The C restatement (knn_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.ko_derive_seed.restype = C.c_uint64
        lib.ko_derive_seed.argtypes = [C.c_uint64] * 4
        lib.ko_mt64_draws.argtypes = [C.c_uint64, _up, C.c_size_t]
        lib.ko_fill_uniform_f64.argtypes = [_dp, C.c_size_t, C.c_uint64]
        lib.ko_fill_uniform_f32.argtypes = [_fp, C.c_size_t, C.c_uint64]
        lib.ko_fill_counter_f32.argtypes = [_fp, C.c_size_t, C.c_size_t, C.c_uint64]
        lib.ko_knn.restype = C.c_int
        lib.ko_knn.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_size_t,
                               C.c_int, C.c_void_p, C.c_int, _ip, _dp]
        lib.ko_knn_f32.restype = C.c_int
        lib.ko_knn_f32.argtypes = [_fp, C.c_size_t, _fp, C.c_size_t, C.c_size_t, C.c_size_t,
                                   C.c_int, C.c_void_p, C.c_int, _ip, _dp]
        lib.ko_pair_distance_f32.restype = C.c_double
        lib.ko_pair_distance_f32.argtypes = [_fp, _fp, C.c_size_t, C.c_int]
        lib.ko_cholesky.restype = C.c_int
        lib.ko_cholesky.argtypes = [_dp, C.c_size_t, _dp]
        lib.ko_whiten.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, _dp]
        lib.ko_max_threads.restype = C.c_int
        self.lib = lib

    # -- inputs ------------------------------------------------------------
    def derive_seed(self, master: int, a: int, b: int = 0, c: int = 0) -> int:
        return int(self.lib.ko_derive_seed(master, a, b, c))

    def mt64_draws(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.lib.ko_mt64_draws(seed, out, count)
        return out

    def uniform_f64(self, n: int, d: int, seed: int) -> np.ndarray:
        out = np.empty((n, d), np.float64)
        self.lib.ko_fill_uniform_f64(out, n * d, seed)
        return out

    def uniform_f32(self, n: int, d: int, seed: int) -> np.ndarray:
        out = np.empty((n, d), np.float32)
        self.lib.ko_fill_uniform_f32(out, n * d, seed)
        return out

    def counter_f32(self, rows: int, d: int, seed: int, row_begin: int = 0) -> np.ndarray:
        out = np.empty((rows, d), np.float32)
        self.lib.ko_fill_counter_f32(out, row_begin * d, rows * d, seed)
        return out

    # -- search ------------------------------------------------------------
    def knn(self, Q, R, k: int, metric: int = EUCLIDEAN, mahal=None, threads: int = 0):
        """bf_knn semantics; Q/R float32 (widened exactly) or float64."""
        n, d = Q.shape
        m = R.shape[0]
        idx = np.empty((n, k), np.int64)
        dist = np.empty((n, k), np.float64)
        mp = None
        if metric == MAHALANOBIS:
            mahal = np.ascontiguousarray(mahal, np.float64)
            mp = mahal.ctypes.data
        if Q.dtype == np.float32:
            s = self.lib.ko_knn_f32(np.ascontiguousarray(Q), n, np.ascontiguousarray(R, np.float32),
                                    m, d, k, metric, mp, threads, idx, dist)
        else:
            s = self.lib.ko_knn(np.ascontiguousarray(Q, np.float64), n,
                                np.ascontiguousarray(R, np.float64), m, d, k, metric, mp,
                                threads, idx, dist)
        if s != 0:
            raise ValueError(f"oracle ko_knn failed with status {s}")
        return idx, dist

    def pair_distance(self, a, b, metric: int = EUCLIDEAN) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return float(self.lib.ko_pair_distance_f32(a, b, a.shape[0], metric))

    def max_threads(self) -> int:
        return int(self.lib.ko_max_threads())


class ReferenceError_(Exception):
    pass


class Reference:
    """The reference's own knn::bf_knn / reference_knn (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference)")
        lib = C.CDLL(path)
        lib.knnref_bf_knn.restype = C.c_int
        lib.knnref_bf_knn.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, C.c_size_t,
                                      C.c_size_t, C.c_int, C.c_void_p, C.c_size_t, C.c_size_t,
                                      C.c_uint, C.c_int, _ip, _dp, C.POINTER(C.c_uint64),
                                      C.c_char_p, C.c_size_t]
        lib.knnref_reference_knn.restype = C.c_int
        lib.knnref_reference_knn.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t,
                                             C.c_size_t, C.c_int, C.c_void_p, _ip, _dp,
                                             C.c_char_p, C.c_size_t]
        lib.knnref_rho_k_all.restype = C.c_int
        lib.knnref_rho_k_all.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp,
                                         C.c_char_p, C.c_size_t]
        lib.knnref_knn_classify.restype = C.c_int
        lib.knnref_knn_classify.argtypes = [_dp, C.c_size_t, C.c_size_t, _ip, C.c_size_t, _dp,
                                            C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, _ip,
                                            C.c_char_p, C.c_size_t]
        lib.knnref_retrieve_vote.restype = C.c_int
        lib.knnref_retrieve_vote.argtypes = [_dp, C.c_size_t, C.c_size_t, _ip, C.c_size_t,
                                             C.c_int64, _dp, C.c_size_t, C.c_size_t, C.c_size_t,
                                             C.c_int, _up, _ip, C.c_char_p, C.c_size_t]
        lib.knnref_derive_seed.restype = C.c_uint64
        lib.knnref_derive_seed.argtypes = [C.c_uint64] * 4
        lib.knnref_uniform.argtypes = [C.c_uint64, _dp, C.c_size_t]
        lib.knnref_mt64_draws.argtypes = [C.c_uint64, _up, C.c_size_t]
        lib.knnref_max_threads.restype = C.c_int
        self.lib = lib

    def bf_knn(self, Q, R, k: int, metric: int = EUCLIDEAN, mahal=None, chunk: int = 1024,
               workers: int = 0, count_evals: bool = False):
        Q = np.ascontiguousarray(Q, np.float64)
        R = np.ascontiguousarray(R, np.float64)
        n, dq = Q.shape
        m, dr = R.shape
        idx = np.empty((n, max(k, 1)), np.int64)
        dist = np.empty((n, max(k, 1)), np.float64)
        evals = C.c_uint64(0)
        err = C.create_string_buffer(512)
        mp, md = None, 0
        if metric == MAHALANOBIS:
            mahal = np.ascontiguousarray(mahal, np.float64)
            mp, md = mahal.ctypes.data, int(round(mahal.size ** 0.5))
        s = self.lib.knnref_bf_knn(Q, n, R, m, dq, dr, k, metric, mp, md, chunk, workers,
                                   int(count_evals), idx, dist, C.byref(evals), err, 512)
        if s == 1:
            raise ValueError(err.value.decode())
        if s != 0:
            raise ReferenceError_(err.value.decode())
        return idx, dist, int(evals.value)

    def reference_knn(self, Q, R, k: int, metric: int = EUCLIDEAN, mahal=None):
        Q = np.ascontiguousarray(Q, np.float64)
        R = np.ascontiguousarray(R, np.float64)
        n, d = Q.shape
        idx = np.empty((n, k), np.int64)
        dist = np.empty((n, k), np.float64)
        err = C.create_string_buffer(512)
        mp = None
        if metric == MAHALANOBIS:
            mahal = np.ascontiguousarray(mahal, np.float64)
            mp = mahal.ctypes.data
        s = self.lib.knnref_reference_knn(Q, n, R, R.shape[0], d, k, metric, mp, idx, dist,
                                          err, 512)
        if s != 0:
            raise ValueError(err.value.decode())
        return idx, dist

    def rho_k_all(self, P, k: int):
        P = np.ascontiguousarray(P, np.float64)
        out = np.empty(P.shape[0], np.float64)
        err = C.create_string_buffer(512)
        if self.lib.knnref_rho_k_all(P, P.shape[0], P.shape[1], k, out, err, 512) != 0:
            raise ValueError(err.value.decode())
        return out

    def knn_classify(self, T, labels, Q, k: int, metric: int = EUCLIDEAN):
        """applications.cpp:36-63 (the reference's own knn_classify)."""
        T = np.ascontiguousarray(T, np.float64)
        Q = np.ascontiguousarray(Q, np.float64)
        lab = np.ascontiguousarray(labels, np.int64)
        out = np.empty(Q.shape[0], np.int64)
        err = C.create_string_buffer(512)
        s = self.lib.knnref_knn_classify(T, T.shape[0], T.shape[1], lab, lab.size, Q, Q.shape[0],
                                         Q.shape[1], k, metric, out, err, 512)
        if s == 1:
            raise ValueError(err.value.decode())
        if s != 0:
            raise ReferenceError_(err.value.decode())
        return out

    def retrieve_vote(self, D, image_of, images: int, Q, k: int, metric: int = EUCLIDEAN):
        """applications.cpp:65-86 (the reference's own retrieve_vote)."""
        D = np.ascontiguousarray(D, np.float64)
        Q = np.ascontiguousarray(Q, np.float64)
        own = np.ascontiguousarray(image_of, np.int64)
        scores = np.empty(max(images, 1), np.uint64)
        ranking = np.empty(max(images, 1), np.int64)
        err = C.create_string_buffer(512)
        s = self.lib.knnref_retrieve_vote(D, D.shape[0], D.shape[1], own, own.size, images, Q,
                                          Q.shape[0], Q.shape[1], k, metric, scores, ranking,
                                          err, 512)
        if s == 1:
            raise ValueError(err.value.decode())
        if s != 0:
            raise ReferenceError_(err.value.decode())
        return scores[:images], ranking[:images]

    def derive_seed(self, master: int, a: int, b: int = 0, c: int = 0) -> int:
        return int(self.lib.knnref_derive_seed(master, a, b, c))

    def uniform(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.float64)
        self.lib.knnref_uniform(seed, out, count)
        return out

    def mt64_draws(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.lib.knnref_mt64_draws(seed, out, count)
        return out

    def max_threads(self) -> int:
        return int(self.lib.knnref_max_threads())


# ----------------------------------------------------------------- comparator
@dataclass
class ParityReport:
    ok: bool
    max_rel: float
    index_mismatches: int
    near_tie_mismatches: int
    bad: list

    def __str__(self):
        return (f"ok={self.ok} max_rel={self.max_rel:.3g} mismatches={self.index_mismatches} "
                f"(near-ties {self.near_tie_mismatches}) bad={self.bad[:5]}")


def compare(gpu_idx, gpu_dist, ref_idx, ref_dist, Q, R, metric: int = EUCLIDEAN,
            rtol: float = 1e-5, oracle: Oracle | None = None, atol: float = 0.0,
            mahal=None) -> ParityReport:
    """North-star tolerance comparator.

    Per query i, rank t: |d_gpu - d_ref| <= rtol * d_ref (+atol for exact
    zeros).  An index mismatch is accepted iff the returned index's distance,
    recomputed in double by the oracle, is within rtol of d_ref[t] (near-tie /
    permutation inside a tie group).  Indices must be distinct and in range.
    """
    gpu_idx = np.asarray(gpu_idx)
    gpu_dist = np.asarray(gpu_dist, np.float64)
    ref_dist = np.asarray(ref_dist, np.float64)
    n, k = ref_idx.shape
    m = R.shape[0]
    bad = []
    tol = rtol * np.abs(ref_dist) + atol
    err = np.abs(gpu_dist - ref_dist)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(ref_dist != 0, err / np.abs(ref_dist), err)
    max_rel = float(rel.max()) if rel.size else 0.0
    for i, t in zip(*np.nonzero(err > tol)):
        bad.append(("dist", int(i), int(t), float(gpu_dist[i, t]), float(ref_dist[i, t])))
    if (gpu_idx < 0).any() or (gpu_idx >= m).any():
        bad.append(("range",))
    for i in range(n):
        if len(np.unique(gpu_idx[i])) != k:
            bad.append(("dup", i))
    mism = np.argwhere(gpu_idx != ref_idx)
    near = 0
    if len(mism):
        oracle = oracle or Oracle()
        Qf = np.ascontiguousarray(Q, np.float32)
        Rf = np.ascontiguousarray(R, np.float32)
        if metric == MAHALANOBIS:
            # recompute on whitened points: y = L^T x (metric.cpp:63-82)
            Mx = np.asarray(mahal, np.float64).reshape(Qf.shape[1], Qf.shape[1])
            L = np.linalg.cholesky(Mx)
            Qf = np.ascontiguousarray(Qf.astype(np.float64) @ L, np.float32)
            Rf = np.ascontiguousarray(Rf.astype(np.float64) @ L, np.float32)
        for i, t in mism:
            j = int(gpu_idx[i, t])
            if not 0 <= j < m:
                continue
            dj = oracle.pair_distance(Qf[i], Rf[j], metric if metric != MAHALANOBIS else 0)
            if abs(dj - ref_dist[i, t]) <= tol[i, t]:
                near += 1
            else:
                bad.append(("idx", int(i), int(t), j, int(ref_idx[i, t]), dj,
                            float(ref_dist[i, t])))
    return ParityReport(ok=not bad, max_rel=max_rel, index_mismatches=len(mism),
                        near_tie_mismatches=near, bad=bad)
