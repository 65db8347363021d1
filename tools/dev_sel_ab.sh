# Dev (GPU): large-k selection A/B (config D shape, k = 100 / 256 / 1024) over
# library variants (args: variant names under build_variants/; "" = in-tree)
for v in "" "$@"; do
  lib=paper_0804_1448_b200/libknn_b200.so; [ -n "$v" ] && lib=build_variants/$v/libknn_b200.so
  echo "=== $lib"
  for k in 100 256 1024; do
    _KNN_B200_DEV_LIB=$lib timeout 120 python tools/prof_shape.py 38400 38400 64 $k 2>&1 | tail -1 | sed 's/.prep_range[^}]*tc_filter_fixed/tc_filter_fixed/; s/, .exact_large_sample.*}//'
  done
done
