"""Generate tests/golden/ fixtures from the REFERENCE itself -- TEST INFRASTRUCTURE.

Runs the reference's own knn::bf_knn (oracle/_ref/libknnref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on small seeded FP32 inputs
(widened exactly to double) and stores inputs + outputs.  The fixtures travel
with the repo so the GPU box (which has no /root/reference) can check parity
against reference outputs.

    python oracle/gen_golden.py        # rewrites tests/golden/*.npz

Cases (paths relative to /root/reference/proj):
  * kat_*      known-answer tests from the reference's suites:
               collinear (tests/test_bruteforce.cpp:77-90), 3-4-5 (test_core.cpp:40-51),
               all-duplicates ties (test_kdtree.cpp:65-75), rho_k line/duplicates
               (test_entropy.cpp:60-72 via bf_knn(points, points, k+1))
  * sweep      acceptance C1-style random instances (tests/acceptance.cpp:58-84):
               n, m <= 200, d <= 32, k <= m, four metrics, uniform [-5, 5)
  * configA    m=n=4800, d=32, k=20 (BASELINE.json configs[0]) -- first 256 queries
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle.oracle import (CHEBYSHEV, EUCLIDEAN, MAHALANOBIS, MANHATTAN, Oracle,  # noqa: E402
                           Reference)

OUT = os.path.join(ROOT, "tests", "golden")
SPD3 = np.array([2.0, 0.4, 0.0, 0.4, 1.5, -0.2, 0.0, -0.2, 1.0])  # acceptance.cpp:60


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    ref = Reference()
    orc = Oracle()
    cases = {}

    def add(name, Q, R, k, metric=EUCLIDEAN, mahal=None):
        Q = np.ascontiguousarray(Q, np.float32)
        R = np.ascontiguousarray(R, np.float32)
        idx, dist, evals = ref.bf_knn(Q, R, k, metric, mahal, count_evals=True)
        cases[name] = dict(Q=Q, R=R, k=np.int64(k), metric=np.int64(metric),
                           mahal=np.asarray(mahal if mahal is not None else [], np.float64),
                           idx=idx, dist=dist, evals=np.uint64(evals))

    # --- known-answer tests ------------------------------------------------
    add("kat_collinear", [[0.1, 0.0]], [[0, 0], [1, 0], [2, 0]], 3)
    add("kat_345", [[0.0, 0.0]], [[3.0, 4.0]], 1)
    add("kat_345_l1", [[0.0, 0.0]], [[3.0, 4.0]], 1, MANHATTAN)
    add("kat_345_linf", [[0.0, 0.0]], [[3.0, 4.0]], 1, CHEBYSHEV)
    add("kat_duplicates", np.full((1, 3), 1.5), np.full((64, 3), 1.5), 5)
    line = np.array([[0.0], [1.0], [3.0]])
    add("kat_rho_line", line, line, 3)
    dup = np.array([[5.0], [5.0], [9.0]])
    add("kat_rho_dup", dup, dup, 2)
    add("kat_mahal_identity", [[1.0, 2.0]], [[4.0, 6.0]], 1, MAHALANOBIS,
        np.array([1.0, 0.0, 0.0, 1.0]))

    # --- acceptance C1-style sweep ------------------------------------------
    rng = np.random.Generator(np.random.PCG64(1001))
    for trial in range(48):
        n = int(rng.integers(1, 201))
        m = int(rng.integers(1, 201))
        metric = trial % 4
        d = 3 if metric == MAHALANOBIS else int(rng.integers(1, 33))
        k = int(rng.integers(1, min(m, 64) + 1))
        Q = orc.uniform_f32(n, d, orc.derive_seed(1001, trial, 1)) * 10 - 5
        R = orc.uniform_f32(m, d, orc.derive_seed(1001, trial, 0)) * 10 - 5
        add(f"sweep_{trial:02d}", Q, R, k, metric, SPD3 if metric == MAHALANOBIS else None)

    # --- configA slice (queries 0..255 of m=n=4800, d=32, k=20) --------------
    R = orc.uniform_f32(4800, 32, orc.derive_seed(42, 4800, 32, 0))
    Q = orc.uniform_f32(4800, 32, orc.derive_seed(42, 4800, 32, 1))[:256]
    add("configA_q256", Q, R, 20)

    flat = {}
    for name, c in cases.items():
        for key, val in c.items():
            flat[f"{name}/{key}"] = val
    np.savez_compressed(os.path.join(OUT, "bf_knn_reference.npz"), **flat)

    # frozen RNG values (tests/test_bench.cpp:44-48) and derive_seed samples
    rngfix = dict(
        uniform_seed1=ref.uniform(1, 2),
        mt64_seed42=ref.mt64_draws(42, 16),
        derive=np.array([ref.derive_seed(42, a, b, c) for a, b, c in
                         [(4800, 32, 0), (4800, 32, 1), (38400, 96, 0), (38400, 96, 1),
                          (19200, 8, 0), (10_000_000, 128, 0)]], np.uint64),
    )
    np.savez_compressed(os.path.join(OUT, "rng_reference.npz"), **rngfix)
    total = sum(os.path.getsize(os.path.join(OUT, f)) for f in os.listdir(OUT))
    print(f"wrote {len(cases)} cases, {total / 1e6:.2f} MB under {OUT}")


if __name__ == "__main__":
    main()
