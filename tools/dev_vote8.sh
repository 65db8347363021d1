# Dev (GPU): fixed-filter per-8-column votes (sparse logs) vs one vote per chunk
for v in "" novote8; do
  lib=paper_0804_1448_b200/libknn_b200.so; [ -n "$v" ] && lib=build_variants/$v/libknn_b200.so
  for sh in "38400 38400 64 33" "38400 38400 64 64" "38400 38400 64 100" "4096 1000000 64 100" "38400 38400 64 1024"; do
    _KNN_B200_DEV_LIB=$lib timeout 120 python tools/prof_shape.py $sh 2>&1 | tail -1 | sed "s#^#[$v] #; s/.prep_range[^}]*tc_filter_fixed/tc_filter_fixed/; s/, .select_large.*//"
  done
done
timeout 600 python -m pytest tests -m gpu -x -q -k "large or every_k or parity" 2>&1 | tail -1
