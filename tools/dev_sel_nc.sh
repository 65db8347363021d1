# Dev (GPU): large-k candidate capacity (KNN_B200_SELECT_NC_MULT) vs fallbacks at low d
for sh in "38400 38400 8 256" "38400 38400 16 1024" "38400 38400 32 256" "38400 38400 64 1024"; do
  for mult in 1 2 4; do
    KNN_B200_SELECT_NC_MULT=$mult timeout 120 python tools/prof_shape.py $sh 2>&1 | tail -1 | sed "s/^/[x$mult] /; s/.prep_range[^}]*tc_filter_fixed/tc_filter_fixed/; s/, .exact_large_sample[^}]*}/}/"
  done
done
