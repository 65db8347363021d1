for lib in paper_0804_1448_b200/libknn_b200.so build_variants/skipkeys/libknn_b200.so; do
  echo "=== lib=$lib"
  _KNN_B200_DEV_LIB=$lib _FM_CHILD=1 timeout 60 python tools/filter_modes.py 38400 38400 96 20 10 2>&1 | grep -o "n=.*total.*" | sed 's/prep[^}]*tc_filter/tc_filter/; s/, .exact_knn.*}//'
  _KNN_B200_DEV_LIB=$lib _FM_CHILD=1 timeout 60 python tools/filter_modes.py 38400 38400 32 20 10 2>&1 | grep -o "n=.*total.*" | sed 's/prep[^}]*tc_filter/tc_filter/; s/, .exact_knn.*}//'
done
