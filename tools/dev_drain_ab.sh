# Dev (GPU): drain batching / buffer capacity A/B on config B and 19200^2 (variant:drain_at pairs)
for vd in ${DRAIN_AB:-"-:8" "bm3:8" "bm7:8" "cap32:8" "cap32:12" "cap32:16" "cap40:16" "cap40:24"}; do
  v=${vd%%:*}; da=${vd##*:}
  lib=paper_0804_1448_b200/libknn_b200.so; [ "$v" != "-" ] && lib=build_variants/$v/libknn_b200.so
  for sh in "38400 38400 96" "19200 19200 96" "19200 19200 8"; do
    KNN_B200_DRAIN_AT=$da _KNN_B200_DEV_LIB=$lib _FM_CHILD=1 timeout 60 python tools/filter_modes.py $sh 20 10 2>&1 | grep -o "n=.*rerank_kernel': [0-9.]*" | sed "s/prep[^}]*tc_filter/tc_filter/; s/^/[$v drain=$da] /"
  done
done
