"""CPU tests of the C ABI boundary: the library loads, exports every symbol the
header declares, and validates arguments exactly like bf_knn
(src/bruteforce.cpp:44-56) -- all host-side, no kernels launched."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "knn_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"KNN_B200_API[^;(]*?\b(knn_b200_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "knn_b200_search" in syms and "knn_b200_merge_device" in syms
    assert len(syms) >= 13


def test_library_exports_every_declared_symbol(knn):
    lib = knn.library()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(knn.EXPORTS) == declared_symbols()


def test_options_struct_layout_matches_header(knn):
    o = knn._Options()
    knn.library().knn_b200_options_init(C.byref(o))
    assert o.struct_size == C.sizeof(knn._Options)
    assert o.chunk_size == 1024 and o.device == -1 and o.path == 0


def test_version(knn):
    assert b"sm_100a" in knn.library().knn_b200_version()


# --- contract errors (host-side validation; no CUDA call happens) -------------
R3 = np.array([[0, 0], [1, 0], [2, 0]], np.float32)
Q1 = np.array([[0.1, 0]], np.float32)


def test_k_exceeds_reference_count(knn):
    with pytest.raises(ValueError, match=r"^bf_knn: k = 4 exceeds reference count 3$"):
        knn.bf_knn(Q1, R3, 4)


def test_k_zero(knn):
    with pytest.raises(ValueError, match=r"^bf_knn: k must be >= 1$"):
        knn.bf_knn(Q1, R3, 0)


def test_dimension_mismatch(knn):
    with pytest.raises(ValueError,
                       match=r"^bf_knn: dimension mismatch, queries have 3, references have 2$"):
        knn.bf_knn(np.zeros((1, 3), np.float32), R3, 1)


def test_chunk_size_zero(knn):
    with pytest.raises(ValueError, match=r"^bf_knn: chunk_size must be >= 1$"):
        knn.bf_knn(Q1, R3, 1, config=knn.BfConfig(chunk_size=0))


def test_validation_order_dim_before_k(knn):
    # bruteforce.cpp:44-49: the dimension check fires before the k check
    with pytest.raises(ValueError, match="dimension mismatch"):
        knn.bf_knn(np.zeros((1, 3), np.float32), R3, 0)


def test_non_finite_coordinate(knn):
    bad = R3.copy()
    bad[1, 1] = np.nan
    with pytest.raises(ValueError, match=r"^PointSet: non-finite coordinate at point 1, dimension 1$"):
        knn.bf_knn(Q1, bad, 1)


def test_mahalanobis_validation(knn):
    with pytest.raises(ValueError, match="not symmetric"):
        knn.bf_knn(Q1, R3, 1, knn.Metric.mahalanobis(2, [1, 0.5, 0.5000001, 1]))
    with pytest.raises(ValueError, match=r"not positive definite \(pivot 1\)"):
        knn.bf_knn(Q1, R3, 1, knn.Metric.mahalanobis(2, [1, 2, 2, 1]))
    with pytest.raises(ValueError, match=r"Mahalanobis matrix is 3x3 but points have dimension 2"):
        knn.bf_knn(Q1, R3, 1, knn.Metric.mahalanobis(3, np.eye(3).ravel()))
    with pytest.raises(ValueError, match="has 3 entries, expected 4"):
        knn.Metric.mahalanobis(2, [1, 0, 0])


def test_merge_argument_validation(knn):
    with pytest.raises(ValueError, match="parts, n and k must be >= 1"):
        knn.merge_device(0, 0, 0, 1, 1, 0, 0)


def test_bf_cost_model_closed_forms():
    """test_bruteforce.cpp:169-181: the paper's operation counts."""
    import math
    import paper_0804_1448_b200 as knn
    unit = knn.bf_cost_model(1, 1, 1, 1)
    assert (unit.additions, unit.multiplications, unit.comparisons) == (2, 1, 0.0)
    c = knn.bf_cost_model(10, 100, 8, 5)
    assert c.multiplications == 8000 and c.additions == 16000
    assert abs(c.comparisons - 1000 * math.log2(100)) < 1e-9
    d = knn.bf_cost_model(10, 100, 16, 5)
    assert d.additions == 2 * c.additions and d.comparisons == c.comparisons
    with pytest.raises(ValueError, match="all inputs must be >= 1"):
        knn.bf_cost_model(0, 1, 1, 1)
