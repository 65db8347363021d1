# dev: per-kernel times on config B (+ config D k=100) and the GPU parity suite
timeout 200 python tools/prof_shape.py 38400 38400 96 20 > gpurun_out/rr.txt 2>&1
timeout 200 python tools/prof_shape.py 38400 38400 96 20 >> gpurun_out/rr.txt 2>&1
timeout 200 python tools/prof_shape.py 38400 38400 64 100 >> gpurun_out/rr.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
