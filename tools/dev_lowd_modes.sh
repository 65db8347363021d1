# Dev (GPU): filter floors (dev modes 0 full / 1 TMEM load + min / 2 no epilogue / 3) at low and high d
for sh in "19200 19200 8" "19200 19200 32" "19200 19200 128" "38400 38400 96"; do
  for mode in 0 1 2 3; do
    KNN_B200_FILTER_MODE=$mode _FM_CHILD=1 _KNN_B200_DEV_LIB=build_variants/devmodes/libknn_b200.so timeout 60 python tools/filter_modes.py $sh 20 5 2>&1 | grep -o "mode=.*rerank_kernel': [0-9.]*" | sed 's/prep[^}]*tc_filter/tc_filter/'
  done
done
