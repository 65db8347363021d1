# dev: e2e vs pipeline chunk size
for c in 65536 32768 19200 12800 9600; do echo "chunk=$c" >> gpurun_out/pipe.txt; KNN_B200_PIPE_CHUNK=$c timeout 200 python tools/e2e_breakdown.py >> gpurun_out/pipe.txt 2>&1; done
