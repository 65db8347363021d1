# Round profile artefacts (run under gpurun): launch list of the bench command
# and one ncu --set full capture per hot kernel of the headline config.
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_under_ncu.log 2>&1
_FM_CHILD=1 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"filter_kernel|rerank_kernel|convert|range_kernel" -s 6 -c 6 \
    -o gpurun_out/full -f python tools/filter_modes.py 38400 38400 96 20 2 > gpurun_out/ncu_full.log 2>&1
