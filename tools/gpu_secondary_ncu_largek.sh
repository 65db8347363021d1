# ncu --set full captures of the large-k kernels only (fixed filter + select at k = 100, select at k = 1024)
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"filter_fixed|select_large" -c 2 -o gpurun_out/sec_large100 -f python tools/prof_shape.py 38400 38400 64 100 >> gpurun_out/ncu_sec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_large" -c 1 -o gpurun_out/sec_large1024 -f python tools/prof_shape.py 38400 38400 64 1024 >> gpurun_out/ncu_sec.log 2>&1
