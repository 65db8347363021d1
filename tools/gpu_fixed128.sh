# dev: large-k filter on d=128 (no-fold) and d=64 (fold) + GPU parity suite
for k in 100 1024; do timeout 120 python tools/prof_shape.py 38400 38400 128 $k >> gpurun_out/fixed128.txt 2>&1; timeout 120 python tools/prof_shape.py 38400 38400 64 $k >> gpurun_out/fixed128.txt 2>&1; done
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
