for c in default 30720 25600 33280 28160,7680 20480,12800 23040,10240,5120; do
  if [ "$c" = default ]; then timeout 120 python tools/e2e_sched.py; else KNN_B200_PIPE_CHUNKS=$c timeout 120 python tools/e2e_sched.py; fi
done
