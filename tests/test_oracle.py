"""CPU tests: pin the C oracle against the reference's golden vectors and the
live reference build (oracle/_ref), so the GPU parity tests can trust it."""
import os

import numpy as np
import pytest

from oracle.oracle import (CHEBYSHEV, EUCLIDEAN, MAHALANOBIS, MANHATTAN, REF_SO, Reference,
                           compare)

HAVE_REF = os.path.exists(REF_SO)


def test_frozen_rng_values(oracle):
    # tests/test_bench.cpp:44-48: first two draws of mt19937_64(1) through the 53-bit map
    v = oracle.uniform_f64(1, 2, 1)
    assert v[0, 0] == 0.13387664401253263
    assert v[0, 1] == 0.13640703636619722


def test_rng_matches_golden(oracle):
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "rng_reference.npz"))
    assert (oracle.uniform_f64(1, 2, 1).ravel() == z["uniform_seed1"]).all()
    assert (oracle.mt64_draws(42, 16) == z["mt64_seed42"]).all()
    got = [oracle.derive_seed(42, a, b, c) for a, b, c in
           [(4800, 32, 0), (4800, 32, 1), (38400, 96, 0), (38400, 96, 1), (19200, 8, 0),
            (10_000_000, 128, 0)]]
    assert (np.array(got, np.uint64) == z["derive"]).all()


def test_fp32_generator_is_exact_and_in_range(oracle):
    x = oracle.uniform_f32(64, 16, 7)
    assert x.dtype == np.float32
    assert (x >= 0).all() and (x < 1).all()
    # (bits >> 40) * 2^-24 == top 24 bits of the same mt19937_64 draws
    bits = oracle.mt64_draws(7, 64 * 16)
    assert (x.ravel() == (bits >> np.uint64(40)).astype(np.float64) * 2.0 ** -24).all()


def test_counter_generator_offsets(oracle):
    full = oracle.counter_f32(100, 8, 99)
    part = oracle.counter_f32(10, 8, 99, row_begin=37)
    assert (full[37:47] == part).all()


def test_oracle_equals_golden_reference_outputs(oracle, golden):
    """Bitwise: the C restatement reproduces the reference's own outputs."""
    for name, c in golden.items():
        metric = int(c["metric"])
        mahal = c["mahal"] if metric == MAHALANOBIS else None
        idx, dist = oracle.knn(c["Q"], c["R"], int(c["k"]), metric, mahal)
        assert (idx == c["idx"]).all(), name
        assert (dist == c["dist"]).all(), name


def test_golden_known_answers(golden):
    # collinear (test_bruteforce.cpp:77-90)
    c = golden["kat_collinear"]
    assert c["idx"].tolist() == [[0, 1, 2]]
    assert np.allclose(c["dist"], [[0.1, 0.9, 1.9]], rtol=1e-6)
    # 3-4-5 triangle (test_core.cpp:40-51)
    assert golden["kat_345"]["dist"][0, 0] == 5.0
    assert golden["kat_345_l1"]["dist"][0, 0] == 7.0
    assert golden["kat_345_linf"]["dist"][0, 0] == 4.0
    # ties at distance zero resolve to the lowest indices (test_kdtree.cpp:65-75)
    assert golden["kat_duplicates"]["idx"].tolist() == [[0, 1, 2, 3, 4]]
    assert (golden["kat_duplicates"]["dist"] == 0).all()
    # rho_k on {0,1,3}: k-th neighbour after the self match (test_entropy.cpp:60-72)
    line = golden["kat_rho_line"]["dist"]
    assert line[0, 1] == 1.0 and line[0, 2] == 3.0 and line[2, 1] == 2.0
    dup = golden["kat_rho_dup"]["dist"]
    assert dup[0, 1] == 0.0 and dup[2, 1] == 4.0


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_oracle_equals_live_reference_random(oracle):
    ref = Reference()
    rng = np.random.default_rng(5)
    spd = np.array([2.0, 0.4, 0.0, 0.4, 1.5, -0.2, 0.0, -0.2, 1.0])
    for trial in range(40):
        metric = trial % 4
        n, m = int(rng.integers(1, 150)), int(rng.integers(1, 150))
        d = 3 if metric == MAHALANOBIS else int(rng.integers(1, 40))
        k = int(rng.integers(1, m + 1))
        Q = (rng.random((n, d)) * 10 - 5).astype(np.float32)
        R = (rng.random((m, d)) * 10 - 5).astype(np.float32)
        if trial % 5 == 0:  # inject exact duplicates to exercise the tie rule
            R[rng.integers(0, m, m // 3)] = R[0]
        mahal = spd if metric == MAHALANOBIS else None
        a = oracle.knn(Q, R, k, metric, mahal)
        b = ref.bf_knn(Q, R, k, metric, mahal)
        c = ref.reference_knn(Q, R, k, metric, mahal)
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
        assert (b[0] == c[0]).all() and (b[1] == c[1]).all()


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_reference_error_texts():
    ref = Reference()
    Q = np.zeros((1, 2))
    R = np.zeros((3, 2))
    with pytest.raises(ValueError, match=r"bf_knn: k = 4 exceeds reference count 3"):
        ref.bf_knn(Q, R, 4)
    with pytest.raises(ValueError, match=r"bf_knn: k must be >= 1"):
        ref.bf_knn(Q, R, 0)
    with pytest.raises(ValueError, match=r"dimension mismatch, queries have 3, references have 2"):
        ref.bf_knn(np.zeros((1, 3)), R, 1)
    with pytest.raises(ValueError, match=r"chunk_size must be >= 1"):
        ref.bf_knn(Q, R, 1, chunk=0)


def test_comparator_accepts_near_ties_and_rejects_errors(oracle):
    R = np.array([[0.0], [1.0], [1.0 + 1e-7], [5.0]], np.float32)
    Q = np.array([[0.5]], np.float32)
    idx, dist = oracle.knn(Q, R, 2)
    # swapped near-tie at rank 1 is accepted
    swapped = idx.copy()
    swapped[0] = [1, 2] if idx[0, 0] == 0 else idx[0]
    rep = compare(idx, dist, idx, dist, Q, R, oracle=oracle)
    assert rep.ok and rep.index_mismatches == 0
    bad = idx.copy()
    bad[0, 1] = 3
    rep = compare(bad, dist, idx, dist, Q, R, oracle=oracle)
    assert not rep.ok
    off = dist.copy()
    off[0, 0] *= 1 + 1e-4
    assert not compare(idx, off, idx, dist, Q, R, oracle=oracle).ok
