# Dev (GPU): cost of a few-query device fallback (margin 2 forces ~1 at k = 100), exact path timing, GPU suite
KNN_B200_LARGE_MARGIN=2 timeout 120 python tools/prof_shape.py 38400 38400 64 100 2>&1 | tail -1
timeout 120 python tools/prof_exact.py 38400 96 20 0 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fb_tests.txt 2>&1; tail -2 gpurun_out/fb_tests.txt
