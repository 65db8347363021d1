# Round bench lines (run under gpurun): default (config B), configs A, C, D, E,
# the exact path on config B, the rho_k self-join, and the reference arm.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_B.json 2> gpurun_out/bench_B.err
for c in A C D E; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --path exact --no-cpu-baseline > gpurun_out/bench_B_exact.json 2> gpurun_out/bench_B_exact.err
timeout 600 python bench.py --task rho_k --no-cpu-baseline > gpurun_out/bench_rho.json 2> gpurun_out/bench_rho.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
