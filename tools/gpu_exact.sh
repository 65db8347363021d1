# dev: exact SIMT path timings (both register budgets) + GPU parity suite
set -x
for minb in 2; do
for a in "38400 96 300 0" "38400 96 512 0" "38400 96 1024 0"; do
  KNN_B200_EXACT_MINB=$minb timeout 120 python tools/prof_exact.py $a >> gpurun_out/exact.txt 2>&1
done
echo "---" >> gpurun_out/exact.txt
done
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
