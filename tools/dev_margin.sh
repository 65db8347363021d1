# Dev (GPU): large-k threshold margin (KNN_B200_LARGE_MARGIN) vs the default, config D shape
for k in 100 256 1024; do
  for mg in default 2 4; do
    if [ $mg = default ]; then timeout 120 python tools/prof_shape.py 38400 38400 64 $k 2>&1 | tail -1 | sed "s/^/[margin=$mg] /; s/.prep_range[^}]*tc_filter_fixed/tc_filter_fixed/";
    else KNN_B200_LARGE_MARGIN=$mg timeout 120 python tools/prof_shape.py 38400 38400 64 $k 2>&1 | tail -1 | sed "s/^/[margin=$mg] /; s/.prep_range[^}]*tc_filter_fixed/tc_filter_fixed/"; fi
  done
done
