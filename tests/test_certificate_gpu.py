"""The tensor path's exactness certificate rests on one
hardware error model: a tcgen05.mma kind::f16 chain over K columns (fp16
operands, fp32 accumulation) computes every element within

    |A - A_exact| <= gamma * sum_c |a_c b_c|,   gamma = (K/16 + 4) * 2^-21,

and the filter's bound uses gamma * (2 ||q~|| max||r~|| + max||r~||^2), which is
>= gamma * sum_c |a_c b_c| by Cauchy-Schwarz.  These tests pin that model with
the certificate's OWN gamma (not a looser one) on adversarial operands --
near-cancelling dot products, magnitudes at the fp16 range limit, mixed
scales, the filter's real operand layout with the folded norm columns -- and
then check end to end that near-tie-saturated data (where the certificate is
at its tightest or must fail) still gives the exact table.

Reference anchors: metric.hpp:22-29 (the key the certificate protects),
topk.cpp:11-33 (the order of the result).
"""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import compare

pytestmark = pytest.mark.gpu

FP16_MAX = 65504.0


def gamma_of(K):
    return (K / 16 + 4) * 2.0 ** -21  # tensor_path.cu: fa.gamma


def _probe(knn, A16, B16):
    import torch
    lib = knn.library()
    fn = lib.knn_b200_debug_mma_probe
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
    K = A16.shape[1]
    dA = torch.from_numpy(A16).cuda()
    dB = torch.from_numpy(B16).cuda()
    dD = torch.empty((128, 128), dtype=torch.float32, device="cuda")
    assert fn(dA.data_ptr(), dB.data_ptr(), K, dD.data_ptr()) == 0
    torch.cuda.synchronize()
    return dD.cpu().numpy().astype(np.float64)


def _operands(kind, K, rng):
    if kind == "uniform":
        A = rng.uniform(-2, 2, (128, K))
        B = rng.uniform(-2, 2, (128, K))
    elif kind == "cancel":
        # every product a_c b_c has a partner -a_c b_c half a row later:
        # exact result 0, sum |ab| large -- all error is accumulation error
        h = K // 2
        U = rng.uniform(-8, 8, (128, h))
        V = rng.uniform(-8, 8, (128, h))
        A = np.concatenate([U, U], 1)
        B = np.concatenate([V, -V], 1)
    elif kind == "partial_cancel":
        h = K // 2
        U = rng.uniform(-8, 8, (128, h))
        V = rng.uniform(-8, 8, (128, h))
        A = np.concatenate([U, U * (1 + rng.uniform(-1e-3, 1e-3, (128, h)))], 1)
        B = np.concatenate([V, -V], 1)
    elif kind == "fp16_range":
        A = rng.choice([-1, 1], (128, K)) * rng.uniform(3e4, FP16_MAX, (128, K))
        B = rng.choice([-1, 1], (128, K)) * rng.uniform(3e4, FP16_MAX, (128, K))
    elif kind == "mixed_scale":
        A = rng.uniform(-1e-3, 1e-3, (128, K))
        B = rng.uniform(-1e-3, 1e-3, (128, K))
        A[:, ::7] = rng.uniform(-1e4, 1e4, (128, A[:, ::7].shape[1]))
        B[:, ::5] = rng.uniform(-1e4, 1e4, (128, B[:, ::5].shape[1]))
    elif kind == "near_tie":
        # many B rows differ from row 0 only in one last-place fp16 bit
        A = rng.uniform(-8, 8, (128, K))
        base = rng.uniform(-8, 8, K).astype(np.float16)
        B16 = np.repeat(base[None, :], 128, 0)
        cols = rng.integers(0, K, 128)
        B16[np.arange(128), cols] = np.nextafter(B16[np.arange(128), cols],
                                                 np.float16(np.inf)).astype(np.float16)
        return A.astype(np.float16), B16
    elif kind == "filter_layout":
        # the filter's operands: r~ in [-8, 8] (fp16), ||r~||^2 split over three
        # fp16 columns; q' = -2 fp16(q~) with 1, 1, 1 in the norm columns
        dd = K - 3
        Rt = rng.uniform(-8, 8, (128, dd)).astype(np.float16).astype(np.float64)
        Qt = rng.uniform(-8, 8, (128, dd)).astype(np.float16).astype(np.float64)
        n2 = (Rt ** 2).sum(1)
        p1 = n2.astype(np.float16).astype(np.float64)
        r1 = n2 - p1
        p2 = r1.astype(np.float16).astype(np.float64)
        p3 = (r1 - p2).astype(np.float16).astype(np.float64)
        B = np.concatenate([Rt, p1[:, None], p2[:, None], p3[:, None]], 1)
        A = np.concatenate([-2 * Qt, np.ones((128, 3))], 1)
    else:
        raise ValueError(kind)
    return A.astype(np.float16), B.astype(np.float16)


KINDS = ["uniform", "cancel", "partial_cancel", "fp16_range", "mixed_scale", "near_tie",
         "filter_layout"]


@pytest.mark.parametrize("K", [16, 32, 64, 96, 112, 128, 144, 256])
@pytest.mark.parametrize("kind", KINDS)
def test_mma_error_within_certificate_gamma(knn, K, kind):
    rng = np.random.default_rng(1000 * K + KINDS.index(kind))
    A16, B16 = _operands(kind, K, rng)
    got = _probe(knn, A16, B16)
    A = A16.astype(np.float64)
    B = B16.astype(np.float64)
    exact = A @ B.T  # fp16 products are exact in double; the sum too at these sizes
    mag = np.abs(A) @ np.abs(B).T
    err = np.abs(got - exact)
    bound = gamma_of(K) * mag
    worst = float((err / np.maximum(bound, 1e-300)).max())
    assert (err <= bound).all(), f"{kind} K={K}: error/bound = {worst:.3f}"
    if kind == "filter_layout":
        # the bound the filter actually uses (Cauchy-Schwarz form) is looser still
        qn = np.sqrt((A[:, :-3] ** 2).sum(1)) / 2
        rn = np.sqrt((B[:, :-3] ** 2).sum(1)).max()
        cs = gamma_of(K) * (2 * qn[:, None] * rn + rn * rn)
        assert (err <= cs).all()


def _check_exact(knn, oracle, Q, R, k):
    t = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_TENSOR))
    fb = knn.last_fallback_count()
    e = knn.bf_knn(Q, R, k, config=knn.BfConfig(path=knn.PATH_EXACT))
    assert (t.index == e.index).all() and (t.distance == e.distance).all()
    ri, rd = oracle.knn(Q, R, k)
    rep = compare(t.index, t.distance, ri, rd, Q, R, oracle=oracle)
    assert rep.ok, rep
    return fb


@pytest.mark.parametrize("spread", [0.0, 1e-7, 1e-5, 1e-4, 3e-4, 1e-3, 1e-2])
def test_sphere_near_ties_are_exact(knn, oracle, spread):
    """References on (nearly) a sphere around every query cluster centre: the
    distances differ by `spread` relative -- from identical (every group is a
    candidate: the logs overflow and the exact kernel takes over) through the
    fp16 resolution (the certificate at its tightest) to well separated."""
    rng = np.random.default_rng(int(spread * 1e7) + 7)
    d, m, k = 32, 12000, 20
    dirs = rng.standard_normal((m, d))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    radii = 1.0 + spread * rng.uniform(0, 1, m)
    R = (0.5 + 0.25 * dirs * radii[:, None]).astype(np.float32)
    Q = (0.5 + 1e-4 * rng.standard_normal((300, d))).astype(np.float32)
    _check_exact(knn, oracle, Q, R, k)


@pytest.mark.parametrize("d", [24, 64, 128])
def test_dense_near_ties_near_fp16_range(knn, oracle, d):
    """Coordinates spanning the fp16 range after centring/scaling, with
    clusters of references that tie to within an ulp (d = 64, 128: the folded
    norms in the narrow 16-wide K block)."""
    rng = np.random.default_rng(11 + d)
    k = 16
    base = rng.uniform(-3e4, 3e4, (400, d)).astype(np.float32)
    R = np.repeat(base, 25, axis=0)
    R += np.float32(1.0) * rng.integers(-1, 2, R.shape).astype(np.float32)
    Q = rng.uniform(-3e4, 3e4, (256, d)).astype(np.float32)
    _check_exact(knn, oracle, Q, R, k)


@pytest.mark.parametrize("d", [16, 128])
def test_queries_far_outside_the_reference_range(knn, oracle, d):
    """a query 4096-8188 reference half-ranges away in two
    coordinates (opposite directions): its scaled coordinate t still rounds to a
    finite fp16 h, but the MMA operand -2 h overflows.  The query must be
    recomputed exactly, never certified on an infinite operand."""
    rng = np.random.default_rng(5)
    m, n, k = 4096, 256, 10
    R = rng.uniform(-1, 1, (m, d)).astype(np.float32)
    Q = rng.uniform(-1, 1, (n, d)).astype(np.float32)
    Q[::3, 0] = 6000.0
    Q[::3, 1] = -7000.0
    Q[1::3, 2] = 5000.0
    Q[1::3, 5] = -8000.0
    fb = _check_exact(knn, oracle, Q, R, k)
    assert fb > 0
