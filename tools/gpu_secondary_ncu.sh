# ncu --set full captures of the secondary paths (exact SIMT kernel, large-k kernels)
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exact_knn -c 1 -o gpurun_out/sec_exact_l2 -f python tools/prof_exact.py 38400 96 20 0 > gpurun_out/ncu_sec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exact_knn -c 1 -o gpurun_out/sec_exact_l1 -f python tools/prof_exact.py 38400 96 20 1 >> gpurun_out/ncu_sec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"filter_fixed|select_large" -c 2 -o gpurun_out/sec_large100 -f python tools/prof_shape.py 38400 38400 64 100 >> gpurun_out/ncu_sec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_large" -c 1 -o gpurun_out/sec_large1024 -f python tools/prof_shape.py 38400 38400 64 1024 >> gpurun_out/ncu_sec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"exact_knn_kernel|select_exact" -s 2 -c 2 -o gpurun_out/sec_exactlarge1024 -f python tools/prof_exact.py 38400 64 1024 1 >> gpurun_out/ncu_sec.log 2>&1
