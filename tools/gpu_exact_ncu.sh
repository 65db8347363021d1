# dev: ncu capture of the exact kernel (config B)
KNN_B200_EXACT_MINB=${MINB:-2} timeout 600 ncu --set full --clock-control none --import-source on -k regex:exact -c 1 -o gpurun_out/exact2 -f python tools/prof_exact.py 38400 96 20 0 > gpurun_out/ncu_exact.log 2>&1
