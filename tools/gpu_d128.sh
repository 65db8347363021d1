# dev: d=128 filter floors (modes 0/2/3) on a config-E-like shape and config C d=128
timeout 300 python tools/filter_modes.py 100000 250000 128 20 2 > gpurun_out/d128.txt 2>&1
timeout 300 python tools/filter_modes.py 19200 19200 128 20 3 >> gpurun_out/d128.txt 2>&1
timeout 300 python tools/filter_modes.py 19200 19200 96 20 3 >> gpurun_out/d128.txt 2>&1
