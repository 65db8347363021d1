# Dev A/B runner (GPU): filter_modes mode 0 (config B) under env variants given as args
for v in "$@"; do
  label=$(echo "$v" | sed 's#[^ ]*/build_variants/\([^/]*\)/[^ ]*#variant:\1#g')
  env $v _FM_CHILD=1 timeout 120 python tools/filter_modes.py 38400 38400 96 20 10 2>&1 | while read -r l; do echo "[$label] $l"; done
done
