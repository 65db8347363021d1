# dev: GPU tests + config-B oracle check + filter timing
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 200 python tools/check_configB.py > gpurun_out/chk.txt 2>&1
timeout 200 python tools/filter_modes.py > gpurun_out/modes.txt 2>&1
