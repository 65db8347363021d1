"""Dev tool (GPU): per-kernel device times of the tensor path on one shape,
optionally under the filter kernel's dev modes (KNN_B200_FILTER_MODE:
0 full, 1 TMEM load + min only, 2 no epilogue work).  Results are only
meaningful for mode 0; the other modes measure floors and need the dev build
(bash tools/build_variant.sh devmodes -DKNN_B200_DEV_MODES, then run with
_KNN_B200_DEV_LIB=build_variants/devmodes/libknn_b200.so).

    python tools/filter_modes.py [n m d k] [reps]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_one(n, m, d, k, reps):
    sys.path.insert(0, ROOT)
    import torch
    import paper_0804_1448_b200 as knn
    Q = torch.empty((n, d), device="cuda")
    R = torch.empty((m, d), device="cuda")
    knn.fill_uniform_device(Q.data_ptr(), n * d, 1)
    knn.fill_uniform_device(R.data_ptr(), m * d, 2)
    od = torch.empty((n, k), device="cuda")
    oi = torch.empty((n, k), dtype=torch.int64, device="cuda")

    def go():
        knn.search_device(Q.data_ptr(), n, R.data_ptr(), m, d, k, od.data_ptr(), oi.data_ptr(),
                          path=knn.PATH_TENSOR)
    go()
    torch.cuda.synchronize()
    knn.profile_enable(True)
    for _ in range(reps):
        go()
    torch.cuda.synchronize()
    prof = knn.profile_collect()
    knn.profile_enable(False)
    # per search: total device time of each kernel name over the reps / reps
    # (a certification retry adds launches of the same kernel names)
    out = {kk: round(v[0] / reps * 1e3, 1) for kk, v in prof.items()}
    print(f"mode={os.environ.get('KNN_B200_FILTER_MODE', '0')} n={n} m={m} d={d} k={k} "
          f"fallbacks={knn.last_fallback_count()} us/search: {out} total {round(sum(out.values()), 1)}",
          flush=True)


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]]
    if os.environ.get("_FM_CHILD"):
        run_one(*args)
    else:
        n, m, d, k = (args + [38400, 38400, 96, 20][len(args):])[:4]
        reps = args[4] if len(args) > 4 else 5
        for mode in (0, 2, 3):
            env = dict(os.environ, KNN_B200_FILTER_MODE=str(mode), _FM_CHILD="1")
            subprocess.run([sys.executable, __file__, str(n), str(m), str(d), str(k),
                            str(reps if mode == 0 else 2)], env=env, check=False)
