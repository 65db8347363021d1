for lib in build_variants/merge32/libknn_b200.so build_variants/bisect/libknn_b200.so build_variants/merge32/libknn_b200.so; do
  echo "=== lib=$lib"
  _KNN_B200_DEV_LIB=$lib bash tools/dev_parts.sh 2>&1 | grep -o "n=.*total.*" | sed 's/prep[^}]*tc_filter/tc_filter/; s/, .exact_knn.*}//'
done
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or certificate or rerank or graph" 2>&1 | tail -3
