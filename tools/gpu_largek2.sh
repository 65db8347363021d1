# dev: large-k timings (both sort networks) + GPU parity suite + filter_fixed ncu
for v in 0 1; do for k in 33 100 256 1024; do KNN_B200_SORT=$v timeout 120 python tools/prof_shape.py 38400 38400 64 $k >> gpurun_out/largek.txt 2>&1; done; echo "--- variant $v" >> gpurun_out/largek.txt; done
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:filter_fixed -c 1 -o gpurun_out/ffix -f python tools/prof_shape.py 38400 38400 64 100 > gpurun_out/ncu_ffix.log 2>&1
