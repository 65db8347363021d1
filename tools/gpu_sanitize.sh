# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_smoke.py
for tool in memcheck synccheck racecheck; do
  timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $tool python tools/sanitize_smoke.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_summary.txt
  tail -3 gpurun_out/san_$tool.txt >> gpurun_out/san_summary.txt
done
