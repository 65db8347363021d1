# Dev (GPU): re-rank candidate staging A/B over the many-part shapes and config B
for lib in paper_0804_1448_b200/libknn_b200.so build_variants/unstaged/libknn_b200.so build_variants/staged8/libknn_b200.so build_variants/staged32/libknn_b200.so; do
  echo "=== lib=$lib"
  _KNN_B200_DEV_LIB=$lib bash tools/dev_parts.sh 2>&1 | grep -o "n=.*total.*" | sed 's/prep[^}]*tc_filter/tc_filter/; s/, .exact_knn.*}//'
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
