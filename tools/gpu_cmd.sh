set -x
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
KNN_B200_FILTER_STATS=1 timeout 120 python tools/filter_modes.py 38400 38400 96 20 2 > gpurun_out/modes.txt 2>&1
timeout 120 python tools/filter_modes.py >> gpurun_out/modes.txt 2>&1
