# Dev (GPU): convert kernel block residency A/B (config B prep times, ncu launch times)
for v in "" cminb5; do
  lib=paper_0804_1448_b200/libknn_b200.so; [ -n "$v" ] && lib=build_variants/$v/libknn_b200.so
  for i in 1 2; do
    _KNN_B200_DEV_LIB=$lib _FM_CHILD=1 timeout 60 python tools/filter_modes.py 38400 38400 96 20 10 2>&1 | grep -o "prep_convert_refs[^,]*, 'prep_convert_queries[^,]*" | sed "s#^#[$v] #"
  done
  _KNN_B200_DEV_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:convert4 -c 6 --csv python tools/prof_shape.py 38400 38400 96 20 2>/dev/null | grep convert4 | awk -F'","' '{print "['"$v"'] ncu", $5, $NF}' | head -6
done
