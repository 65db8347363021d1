# Dev (GPU): config A filter floors (dev modes 0 / 2 / 3) and per-kernel times
for mode in 0 2 3; do
  KNN_B200_FILTER_MODE=$mode _FM_CHILD=1 _KNN_B200_DEV_LIB=build_variants/devmodes/libknn_b200.so timeout 60 python tools/filter_modes.py 4800 4800 32 20 10 2>&1 | grep -o "mode=.*"
done
