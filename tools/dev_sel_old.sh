# Dev (GPU): low-d large-k fallbacks, current vs the pre-round-2-select build
for lib in paper_0804_1448_b200/libknn_b200.so build_variants/oldsel/libknn_b200.so; do
  for sh in "38400 38400 8 256" "38400 38400 16 1024" "38400 38400 32 256" "38400 38400 8 100"; do
    _KNN_B200_DEV_LIB=$lib timeout 120 python tools/prof_shape.py $sh 2>&1 | tail -1 | sed "s#^#[$lib] #; s/.prep_range[^}]*tc_filter_fixed/tc_filter_fixed/; s/, .exact_large_sample[^}]*}/}/"
  done
done
