# Dev (GPU): filter + re-rank on shapes with many stream-K parts per query
for sh in "4800 4800 32" "2560 40000 64" "1024 100000 96" "19200 19200 96" "38400 38400 96"; do
  _FM_CHILD=1 timeout 60 python tools/filter_modes.py $sh 20 10
done
