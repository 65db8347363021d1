# Dev (GPU): fixed-filter vote skip (KNN_B200_LOG_ALL) at config D's large k
for k in 33 100 256 1024; do
  for la in 0 1; do
    KNN_B200_LOG_ALL=$la timeout 120 python tools/prof_shape.py 38400 38400 64 $k 2>&1 | tail -1 | sed "s/^/[log_all=$la] /; s/.prep_range[^}]*tc_filter_fixed/tc_filter_fixed/; s/, .select_large.*//"
  done
done
timeout 120 python tools/prof_shape.py 1024 1000000 64 100 2>&1 | tail -1 | sed "s/.prep_range[^}]*tc_filter_fixed/tc_filter_fixed/; s/, .select_large.*//"
