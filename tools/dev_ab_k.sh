# Dev A/B runner (GPU): config D shape at k = $1 under env variants given as further args
k=$1; shift
for v in "$@"; do
  env $v _FM_CHILD=1 timeout 120 python tools/filter_modes.py 38400 38400 64 $k 3 2>&1 | sed "s/^/[$v] /"
done
