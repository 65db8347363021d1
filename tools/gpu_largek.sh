# dev: per-kernel times of the large-k tensor path (config D) + ncu of the select kernel
for k in 100 256 1024; do timeout 120 python tools/prof_shape.py 38400 38400 64 $k >> gpurun_out/largek.txt 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_large -c 1 -o gpurun_out/sel1024 -f python tools/prof_shape.py 38400 38400 64 1024 > gpurun_out/ncu_sel.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_large -c 1 -o gpurun_out/sel100 -f python tools/prof_shape.py 38400 38400 64 100 >> gpurun_out/ncu_sel.log 2>&1
