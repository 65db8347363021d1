# dev: tests, modes, and ncu captures of the rerank + prep kernels
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 200 python tools/filter_modes.py > gpurun_out/modes.txt 2>&1
_FM_CHILD=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rerank|convert|range" -s 4 -c 4 -o gpurun_out/rr -f python tools/filter_modes.py 38400 38400 96 20 2 > gpurun_out/ncu_rr.log 2>&1
