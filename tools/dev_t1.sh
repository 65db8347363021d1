# dev: GPU parity suite + config-B filter timing (run under gpurun)
python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3 > gpurun_out/t1_tests.txt
for i in 1 2; do _FM_CHILD=1 python tools/filter_modes.py 38400 38400 96 20 10 ; done > gpurun_out/t1_time.txt 2>&1
