# Dev (GPU): re-rank A/B over library variants (args: variant names under build_variants/)
for v in "" "$@"; do
  lib=paper_0804_1448_b200/libknn_b200.so; [ -n "$v" ] && lib=build_variants/$v/libknn_b200.so
  echo "=== $lib"
  for sh in "38400 38400 96" "38400 38400 32" "19200 19200 96" "19200 19200 8" "4800 4800 32"; do
    _KNN_B200_DEV_LIB=$lib _FM_CHILD=1 timeout 60 python tools/filter_modes.py $sh 20 10 2>&1 | grep -o "n=.*total.*" | sed 's/prep[^}]*tc_filter/tc_filter/; s/, .exact_knn.*}//'
  done
done
