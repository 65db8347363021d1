# Dev A/B runner (GPU): filter_modes mode 0 under env variants given as args
for v in "$@"; do
  env $v _FM_CHILD=1 timeout 120 python tools/filter_modes.py 38400 38400 96 20 10 2>&1 | sed "s/^/[$v] /"
done
