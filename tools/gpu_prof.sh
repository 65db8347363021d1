# dev: modes + one ncu --set full capture of the mode-0 filter kernel
timeout 200 python tools/filter_modes.py > gpurun_out/modes.txt 2>&1
_FM_CHILD=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:filter_kernel -s 1 -c 1 -o gpurun_out/filt -f python tools/filter_modes.py 38400 38400 96 20 2 > gpurun_out/ncu.log 2>&1
