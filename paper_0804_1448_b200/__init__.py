"""B200-native brute-force kNN engine (drop-in for the reference's ``knn::bf_knn``).

Python host mirror of the reference's operator interface for the hot path
(``/root/reference/proj/include/knn/bruteforce.hpp:12-33``): ``BfConfig``,
``SearchStats``, ``Metric`` and ``bf_knn(queries, references, k, metric,
config, stats)`` with the same argument meaning, output ordering and error
behaviour (``ValueError`` where the reference throws
``std::invalid_argument``, with the same message text).  Every call goes
through the C ABI of ``libknn_b200.so`` (``include/knn_b200.h``); there is no
CPU fallback -- if the CUDA library is missing or no GPU is present the calls
raise ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "BfConfig", "SearchStats", "Metric", "NeighborTable", "bf_knn", "search_device",
    "Index", "merge_device", "library", "lib_path", "KnnError", "PATH_AUTO", "PATH_EXACT",
    "PATH_TENSOR", "launch_count", "reset_launch_count", "profile_enable", "profile_collect",
    "fill_uniform_device", "Sharded", "Comm", "rho_k_all", "knn_classify", "retrieve_vote",
    "VoteTally", "nccl_unique_id", "SHARD_REFERENCES",
    "SHARD_QUERIES",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libknn_b200.so")
# dev-only: A/B builds of the same library (tools/build_variant.sh)
lib_path = os.environ.get("_KNN_B200_DEV_LIB", lib_path)

EUCLIDEAN, MANHATTAN, CHEBYSHEV, MAHALANOBIS = 0, 1, 2, 3
PATH_AUTO, PATH_EXACT, PATH_TENSOR = 0, 1, 2
_STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENCCL", 5: "EINTERNAL"}

EXPORTS = [
    "knn_b200_options_init", "knn_b200_last_error", "knn_b200_version", "knn_b200_search",
    "knn_b200_search_device", "knn_b200_index_create", "knn_b200_index_create_device",
    "knn_b200_index_search", "knn_b200_index_search_device", "knn_b200_index_destroy",
    "knn_b200_merge_device", "knn_b200_launch_count", "knn_b200_reset_launch_count",
    "knn_b200_profile_enable", "knn_b200_profile_only", "knn_b200_profile_collect", "knn_b200_fill_uniform_device",
    "knn_b200_last_fallback_count", "knn_b200_debug_mma_probe",
    "knn_b200_sharded_create", "knn_b200_sharded_search", "knn_b200_sharded_destroy",
    "knn_b200_nccl_unique_id", "knn_b200_nccl_version", "knn_b200_comm_create",
    "knn_b200_comm_destroy", "knn_b200_dist_search_device", "knn_b200_rho_k_all",
    "knn_b200_rho_k_all_device", "knn_b200_knn_classify", "knn_b200_retrieve_vote",
]
SHARD_REFERENCES, SHARD_QUERIES = 0, 1


class KnnError(RuntimeError):
    """A device-side failure (ENOMEM / ECUDA / ENCCL / EINTERNAL)."""

    def __init__(self, status: int, message: str):
        super().__init__(f"knn_b200 {_STATUS.get(status, status)}: {message}")
        self.status = status


class _Options(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32),
        ("device", C.c_int32),
        ("path", C.c_int32),
        ("count_distance_evals", C.c_int32),
        ("chunk_size", C.c_uint64),
        ("worker_count", C.c_uint32),
        ("raw_keys", C.c_int32),
        ("mahalanobis", C.c_void_p),
        ("mahalanobis_dim", C.c_int64),
        ("stream", C.c_void_p),
    ]


_lib = None


def library() -> C.CDLL:
    """Load libknn_b200.so (built by ``__graft_entry__.build()``); fail loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise RuntimeError(f"{lib_path} is missing: run `python -c 'import __graft_entry__ as g; "
                           "g.build()'` (there is no CPU fallback)")
    # NCCL is loaded by the library at first use: point it at the pip NCCL that
    # PyTorch links (if present), so both share one libnccl.so.2 in the process
    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep NCCL's banner off stdout (bench JSON)
    if "KNN_B200_NCCL_LIB" not in os.environ:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        if spec is not None and spec.submodule_search_locations:
            cand = os.path.join(list(spec.submodule_search_locations)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["KNN_B200_NCCL_LIB"] = cand
    lib = C.CDLL(lib_path)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    lib.knn_b200_options_init.argtypes = [C.POINTER(_Options)]
    lib.knn_b200_last_error.restype = C.c_char_p
    lib.knn_b200_version.restype = C.c_char_p
    lib.knn_b200_search.argtypes = [vp, i64, i32, vp, i64, i32, i32, i32, C.POINTER(_Options),
                                    vp, vp, C.POINTER(C.c_uint64)]
    lib.knn_b200_search_device.argtypes = [vp, i64, vp, i64, i32, i32, i32, C.POINTER(_Options),
                                           vp, vp]
    lib.knn_b200_index_create.argtypes = [vp, i64, i32, i64, C.POINTER(_Options),
                                          C.POINTER(vp)]
    lib.knn_b200_index_create_device.argtypes = [vp, i64, i32, i64, C.POINTER(_Options),
                                                 C.POINTER(vp)]
    lib.knn_b200_index_search.argtypes = [vp, vp, i64, i32, i32, C.POINTER(_Options), vp, vp]
    lib.knn_b200_index_search_device.argtypes = [vp, vp, i64, i32, i32, C.POINTER(_Options),
                                                 vp, vp]
    lib.knn_b200_index_destroy.argtypes = [vp]
    lib.knn_b200_merge_device.argtypes = [vp, vp, i32, i64, i32, i32, vp, vp, vp]
    lib.knn_b200_launch_count.restype = C.c_uint64
    lib.knn_b200_profile_enable.argtypes = [C.c_int]
    lib.knn_b200_profile_only.argtypes = [C.c_char_p]
    lib.knn_b200_profile_collect.restype = C.c_int
    lib.knn_b200_profile_collect.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_double),
                                             C.POINTER(C.c_uint64), C.c_int]
    lib.knn_b200_last_fallback_count.restype = C.c_int
    lib.knn_b200_last_fallback_count.argtypes = [C.c_int]
    lib.knn_b200_fill_uniform_device.restype = C.c_int
    lib.knn_b200_fill_uniform_device.argtypes = [vp, i64, C.c_uint64, i64, vp]
    lib.knn_b200_sharded_create.argtypes = [vp, i64, i32, i32, vp, i32, C.POINTER(_Options),
                                            C.POINTER(vp)]
    lib.knn_b200_sharded_search.argtypes = [vp, vp, i64, i32, i32, C.POINTER(_Options), vp, vp]
    lib.knn_b200_sharded_destroy.argtypes = [vp]
    lib.knn_b200_nccl_unique_id.argtypes = [vp, C.c_size_t]
    lib.knn_b200_nccl_version.restype = C.c_int
    lib.knn_b200_comm_create.argtypes = [vp, C.c_size_t, i32, i32, i32, C.POINTER(vp)]
    lib.knn_b200_comm_destroy.argtypes = [vp]
    lib.knn_b200_dist_search_device.argtypes = [vp, vp, vp, i64, i32, i32, C.POINTER(_Options),
                                                vp, vp]
    lib.knn_b200_rho_k_all.argtypes = [vp, i64, i32, i32, C.POINTER(_Options), vp]
    lib.knn_b200_rho_k_all_device.argtypes = [vp, i64, i32, i32, C.POINTER(_Options), vp]
    lib.knn_b200_knn_classify.argtypes = [vp, i64, i32, vp, vp, i64, i32, i32, i32,
                                          C.POINTER(_Options), vp]
    lib.knn_b200_retrieve_vote.argtypes = [vp, i64, i32, vp, i64, vp, i64, i32, i32, i32,
                                           C.POINTER(_Options), vp, vp]
    for name in ("knn_b200_rho_k_all", "knn_b200_rho_k_all_device", "knn_b200_knn_classify",
                 "knn_b200_retrieve_vote"):
        getattr(lib, name).restype = C.c_int
    for name in ("knn_b200_search", "knn_b200_search_device", "knn_b200_index_create",
                 "knn_b200_index_create_device", "knn_b200_index_search",
                 "knn_b200_index_search_device", "knn_b200_merge_device",
                 "knn_b200_sharded_create", "knn_b200_sharded_search",
                 "knn_b200_nccl_unique_id", "knn_b200_comm_create",
                 "knn_b200_dist_search_device"):
        getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def launch_count() -> int:
    return int(library().knn_b200_launch_count())


def reset_launch_count() -> None:
    library().knn_b200_reset_launch_count()


def last_fallback_count(device: int = -1) -> int:
    """Queries of the last tensor-path search that failed certification."""
    return int(library().knn_b200_last_fallback_count(device))


def profile_enable(on: bool = True, only: str = "") -> None:
    """Bracket every engine launch on this thread (or only those whose name
    starts with `only`) with CUDA events."""
    library().knn_b200_profile_only(only.encode())
    library().knn_b200_profile_enable(int(bool(on)))


def profile_collect() -> dict:
    """{kernel name: (total ms, launches)} since the last collect (synchronizes)."""
    names = C.create_string_buffer(4096)
    ms = (C.c_double * 64)()
    cnt = (C.c_uint64 * 64)()
    nk = library().knn_b200_profile_collect(names, 4096, ms, cnt, 64)
    if nk < 0:
        raise KnnError(3, "profile_collect: event synchronization failed")
    keys = [x for x in names.value.decode().split("\n") if x]
    return {keys[i]: (ms[i], int(cnt[i])) for i in range(min(nk, len(keys)))}


def fill_uniform_device(ptr: int, count: int, seed: int, offset: int = 0,
                        stream: int = 0) -> None:
    """Device-side synthetic uniform [0,1) FP32 (splitmix64 counter stream)."""
    _check(library().knn_b200_fill_uniform_device(ptr, count, seed, offset, stream or None))


def _check(status: int) -> None:
    if status == 0:
        return
    msg = library().knn_b200_last_error().decode()
    if status == 1:
        raise ValueError(msg)
    raise KnnError(status, msg)


NCCL_ID_BYTES = 128


# --------------------------------------------------------------- mirror types
@dataclass
class BfConfig:
    """bruteforce.hpp:12-20.  chunk_size / worker_count never change results."""
    chunk_size: int = 1024
    worker_count: int = 0
    count_distance_evals: bool = False
    path: int = PATH_AUTO      # engine extension: which device path computes the keys
    device: int = -1


@dataclass
class SearchStats:
    """bruteforce.hpp:22-25."""
    distance_evals: int = 0
    pruned_subtrees: int = 0


@dataclass
class Metric:
    """metric.hpp:52-106 (kind + optional Mahalanobis inverse covariance)."""
    kind: int = EUCLIDEAN
    matrix: Optional[np.ndarray] = field(default=None, repr=False)

    @staticmethod
    def euclidean() -> "Metric":
        return Metric(EUCLIDEAN)

    @staticmethod
    def manhattan() -> "Metric":
        return Metric(MANHATTAN)

    @staticmethod
    def chebyshev() -> "Metric":
        return Metric(CHEBYSHEV)

    @staticmethod
    def mahalanobis(d: int, matrix) -> "Metric":
        m = np.ascontiguousarray(np.asarray(matrix, np.float64).reshape(-1))
        if m.size != d * d:
            raise ValueError(f"Metric: Mahalanobis matrix has {m.size} entries, expected {d * d}")
        return Metric(MAHALANOBIS, m)


@dataclass
class NeighborTable:
    """neighbor_table.hpp:22-44 as SoA arrays: ``index`` int64 (n, k) and
    ``distance`` (n, k), row-major by query, ascending, ties by index."""
    index: np.ndarray
    distance: np.ndarray

    @property
    def query_count(self) -> int:
        return self.index.shape[0]

    @property
    def k(self) -> int:
        return self.index.shape[1]

    def row(self, i: int):
        return list(zip(self.index[i].tolist(), self.distance[i].tolist()))


def _opts(config: Optional[BfConfig] = None, metric: Optional[Metric] = None,
          raw_keys: bool = False, stream: int = 0) -> _Options:
    o = _Options()
    library().knn_b200_options_init(C.byref(o))
    if config is not None:
        o.chunk_size = int(config.chunk_size)
        o.worker_count = int(config.worker_count)
        o.count_distance_evals = int(bool(config.count_distance_evals))
        o.path = int(config.path)
        o.device = int(config.device)
    o.raw_keys = int(raw_keys)
    o.stream = stream or None
    return o


def _as_points(x) -> np.ndarray:
    a = np.asarray(x)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    return np.ascontiguousarray(a, dtype=np.float32)


def bf_knn(queries, references, k: int, metric: Metric = None, config: BfConfig = None,
           stats: SearchStats = None, out=None) -> NeighborTable:
    """Exhaustive exact kNN on the GPU (bruteforce.hpp:31-33 semantics).

    ``queries`` (n, d) and ``references`` (m, d) are host arrays (narrowed to
    float32).  Returns a NeighborTable with float32 distances (sqrt'd for
    euclidean / mahalanobis) and int64 indices.
    """
    metric = metric or Metric.euclidean()
    config = config or BfConfig()
    lib = library()
    Q = _as_points(queries)
    R = _as_points(references)
    n, dq = Q.shape
    m, dr = R.shape
    kk = max(int(k), 0)
    if out is not None:  # caller-provided (e.g. pinned) output arrays
        out_d, out_i = out
        if out_d.shape != (n, kk) or out_i.shape != (n, kk) or out_d.dtype != np.float32 \
                or out_i.dtype != np.int64 or not out_d.flags.c_contiguous \
                or not out_i.flags.c_contiguous:
            raise ValueError("bf_knn: out arrays must be C-contiguous (n, k) float32 / int64")
    else:
        out_d = np.empty((n, max(kk, 1)), np.float32)
        out_i = np.empty((n, max(kk, 1)), np.int64)
    o = _opts(config, metric)
    keep = None
    if metric.kind == MAHALANOBIS:
        keep = np.ascontiguousarray(metric.matrix, np.float64)
        o.mahalanobis = keep.ctypes.data
        o.mahalanobis_dim = int(round(keep.size ** 0.5))
    evals = C.c_uint64(0)
    _check(lib.knn_b200_search(Q.ctypes.data, n, dq, R.ctypes.data, m, dr, int(k), metric.kind,
                               C.byref(o), out_d.ctypes.data, out_i.ctypes.data, C.byref(evals)))
    if stats is not None:
        stats.distance_evals = int(evals.value)
    return NeighborTable(out_i, out_d)


@dataclass
class BfCostModel:
    """bruteforce.hpp:35-43: the paper's closed-form operation counts."""
    additions: int
    multiplications: int
    comparisons: float


def bf_cost_model(n: int, m: int, d: int, k: int) -> BfCostModel:
    """bruteforce.cpp:102-112: adds 2nmd, muls nmd, comparisons n m log2 m."""
    if n <= 0 or m <= 0 or d <= 0 or k <= 0:
        raise ValueError("bf_cost_model: all inputs must be >= 1")
    nmd = n * m * d
    return BfCostModel(2 * nmd, nmd, float(n) * float(m) * math.log2(float(m)))


def search_device(q_ptr: int, n: int, r_ptr: int, m: int, d: int, k: int, out_dist_ptr: int,
                  out_idx_ptr: int, metric: int = EUCLIDEAN, path: int = PATH_AUTO,
                  stream: int = 0, raw_keys: bool = False, device: int = -1,
                  mahalanobis=None) -> None:
    """Device-resident search on raw device pointers (e.g. ``tensor.data_ptr()``).
    ``mahalanobis``: the d x d matrix when ``metric`` is MAHALANOBIS (the
    inputs are whitened on the device into scratch copies)."""
    cfg = BfConfig(path=path, device=device)
    o = _opts(cfg, raw_keys=raw_keys, stream=stream)
    keep = None
    if mahalanobis is not None:
        keep = np.ascontiguousarray(mahalanobis, np.float64)
        o.mahalanobis = keep.ctypes.data
        o.mahalanobis_dim = int(round(keep.size ** 0.5))
    _check(library().knn_b200_search_device(q_ptr, n, r_ptr, m, d, k, metric, C.byref(o),
                                            out_dist_ptr, out_idx_ptr))


def merge_device(part_keys_ptr: int, part_idx_ptr: int, parts: int, n: int, k: int,
                 out_dist_ptr: int, out_idx_ptr: int, metric: int = EUCLIDEAN,
                 stream: int = 0) -> None:
    """Merge parts x n x k raw-key lists (sorted per part) into finalized top-k."""
    _check(library().knn_b200_merge_device(part_keys_ptr, part_idx_ptr, parts, n, k, metric,
                                           stream or None, out_dist_ptr, out_idx_ptr))


class Index:
    """Device-resident reference set (build once, search many; kdtree.hpp:21,70-72 split)."""

    def __init__(self, references=None, *, device_ptr: int = 0, m: int = 0, d: int = 0,
                 index_base: int = 0, device: int = -1):
        lib = library()
        h = C.c_void_p()
        o = _opts(BfConfig(device=device))
        if device_ptr:
            _check(lib.knn_b200_index_create_device(device_ptr, m, d, index_base, C.byref(o),
                                                    C.byref(h)))
            self.m, self.d = m, d
        else:
            R = _as_points(references)
            self.m, self.d = R.shape
            _check(lib.knn_b200_index_create(R.ctypes.data, self.m, self.d, index_base,
                                             C.byref(o), C.byref(h)))
        self._h = h
        self.index_base = index_base

    def search(self, queries, k: int, metric: int = EUCLIDEAN, path: int = PATH_AUTO,
               raw_keys: bool = False) -> NeighborTable:
        Q = _as_points(queries)
        n = Q.shape[0]
        out_d = np.empty((n, k), np.float32)
        out_i = np.empty((n, k), np.int64)
        o = _opts(BfConfig(path=path), raw_keys=raw_keys)
        _check(library().knn_b200_index_search(self._h, Q.ctypes.data, n, k, metric, C.byref(o),
                                               out_d.ctypes.data, out_i.ctypes.data))
        return NeighborTable(out_i, out_d)

    def search_device(self, q_ptr: int, n: int, k: int, out_dist_ptr: int, out_idx_ptr: int,
                      metric: int = EUCLIDEAN, path: int = PATH_AUTO, stream: int = 0,
                      raw_keys: bool = False) -> None:
        o = _opts(BfConfig(path=path), raw_keys=raw_keys, stream=stream)
        _check(library().knn_b200_index_search_device(self._h, q_ptr, n, k, metric, C.byref(o),
                                                      out_dist_ptr, out_idx_ptr))

    def close(self) -> None:
        if self._h:
            library().knn_b200_index_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Sharded:
    """One process, several GPUs: the reference set split into
    contiguous shards (``mode=SHARD_REFERENCES``: per-device top-k, NCCL
    all-gather, device merge -- bitwise one search over all of R) or the
    queries split over devices that each hold all of R (``SHARD_QUERIES``)."""

    def __init__(self, references, num_devices: int, mode: int = SHARD_REFERENCES,
                 devices=None):
        R = _as_points(references)
        self.m, self.d = R.shape
        self.num_devices = int(num_devices)
        h = C.c_void_p()
        devs = None
        if devices is not None:
            devs = (C.c_int32 * len(devices))(*devices)
        o = _opts()
        _check(library().knn_b200_sharded_create(R.ctypes.data, self.m, self.d, self.num_devices,
                                                 C.cast(devs, C.c_void_p) if devs else None,
                                                 int(mode), C.byref(o), C.byref(h)))
        self._h = h

    def search(self, queries, k: int, metric: int = EUCLIDEAN,
               path: int = PATH_AUTO) -> NeighborTable:
        Q = _as_points(queries)
        n = Q.shape[0]
        out_d = np.empty((n, k), np.float32)
        out_i = np.empty((n, k), np.int64)
        o = _opts(BfConfig(path=path))
        _check(library().knn_b200_sharded_search(self._h, Q.ctypes.data, n, int(k), metric,
                                                 C.byref(o), out_d.ctypes.data,
                                                 out_i.ctypes.data))
        return NeighborTable(out_i, out_d)

    def close(self) -> None:
        if self._h:
            library().knn_b200_sharded_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 creates it; the caller broadcasts it)."""
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _check(library().knn_b200_nccl_unique_id(buf, NCCL_ID_BYTES))
    return buf.raw


class Comm:
    """One rank of a one-process-per-GPU job (e.g. under torchrun): the NCCL
    communicator the reference-sharded search all-gathers over."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int, device: int):
        if len(unique_id) < NCCL_ID_BYTES:
            raise ValueError("Comm: unique id must hold 128 bytes")
        buf = C.create_string_buffer(bytes(unique_id[:NCCL_ID_BYTES]), NCCL_ID_BYTES)
        h = C.c_void_p()
        _check(library().knn_b200_comm_create(buf, NCCL_ID_BYTES, nranks, rank, device,
                                              C.byref(h)))
        self._h = h
        self.nranks, self.rank, self.device = nranks, rank, device

    def search_device(self, shard: "Index", q_ptr: int, n: int, k: int, out_dist_ptr: int,
                      out_idx_ptr: int, metric: int = EUCLIDEAN, path: int = PATH_AUTO,
                      stream: int = 0) -> None:
        """This rank's shard search + NCCL all-gather + device merge: every rank
        receives the final n x k table over all shards."""
        o = _opts(BfConfig(path=path), stream=stream)
        _check(library().knn_b200_dist_search_device(self._h, shard._h, q_ptr, n, int(k), metric,
                                                     C.byref(o), out_dist_ptr, out_idx_ptr))

    def close(self) -> None:
        if self._h:
            library().knn_b200_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_version() -> int:
    return int(library().knn_b200_nccl_version())


# ------------------------------------------------ callers of the hot path ----
def rho_k_all(points, k: int, config: BfConfig = None) -> np.ndarray:
    """entropy.cpp:75-89: distance from every point to its k-th nearest other
    point (self excluded by index), one device self-join + epilogue."""
    P = _as_points(points)
    n, d = P.shape
    out = np.empty(n, np.float64)
    o = _opts(config)
    _check(library().knn_b200_rho_k_all(P.ctypes.data, n, d, int(k), C.byref(o), out.ctypes.data))
    return out


def rho_k_all_device(points_ptr: int, n: int, d: int, k: int, out_ptr: int,
                     stream: int = 0) -> None:
    """Device pointers: float32 n x d points in, float64 n distances out."""
    o = _opts(stream=stream)
    _check(library().knn_b200_rho_k_all_device(points_ptr, n, d, int(k), C.byref(o), out_ptr))


def knn_classify(train_points, labels, queries, k: int, metric: Metric = None,
                 config: BfConfig = None) -> np.ndarray:
    """applications.cpp:36-63 (LabeledSet = train_points + labels)."""
    T = _as_points(train_points)
    Q = _as_points(queries)
    lab = np.ascontiguousarray(labels, np.int64)
    if lab.size != T.shape[0]:
        raise ValueError(f"LabeledSet: {lab.size} labels for {T.shape[0]} points")
    metric = metric or Metric.euclidean()
    if metric.kind == MAHALANOBIS:
        raise ValueError("knn_classify: use bf_knn for the Mahalanobis metric")
    out = np.empty(Q.shape[0], np.int64)
    o = _opts(config)
    _check(library().knn_b200_knn_classify(T.ctypes.data, T.shape[0], T.shape[1], lab.ctypes.data,
                                           Q.ctypes.data, Q.shape[0], Q.shape[1], int(k),
                                           metric.kind, C.byref(o), out.ctypes.data))
    return out


@dataclass
class VoteTally:
    """applications.hpp: per-image vote counts and the ranking."""
    scores: np.ndarray
    ranking: np.ndarray


def retrieve_vote(descriptors, image_of, image_count: int, query_descriptors, k: int,
                  metric: Metric = None, config: BfConfig = None) -> VoteTally:
    """applications.cpp:65-86 (DescriptorDatabase = descriptors + image_of)."""
    D = _as_points(descriptors)
    Q = _as_points(query_descriptors)
    own = np.ascontiguousarray(image_of, np.int64)
    if own.size != D.shape[0]:
        raise ValueError(f"DescriptorDatabase: {own.size} owners for {D.shape[0]} descriptors")
    metric = metric or Metric.euclidean()
    if metric.kind == MAHALANOBIS:
        raise ValueError("retrieve_vote: use bf_knn for the Mahalanobis metric")
    ic = int(image_count)
    scores = np.empty(max(ic, 1), np.uint64)
    ranking = np.empty(max(ic, 1), np.int64)
    o = _opts(config)
    _check(library().knn_b200_retrieve_vote(D.ctypes.data, D.shape[0], D.shape[1], own.ctypes.data,
                                            ic, Q.ctypes.data, Q.shape[0], Q.shape[1], int(k),
                                            metric.kind, C.byref(o), scores.ctypes.data,
                                            ranking.ctypes.data))
    return VoteTally(scores[:ic], ranking[:ic])
