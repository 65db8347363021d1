# Dev (GPU): CTAs per query-tile pair cap (KNN_B200_CTAS_PER_PAIR) on small query sets
for cap in 29 8 6 4 3; do
  for sh in "4800 4800 32" "2560 40000 64" "4800 38400 96"; do
    KNN_B200_CTAS_PER_PAIR=$cap _FM_CHILD=1 timeout 60 python tools/filter_modes.py $sh 20 10 2>&1 | grep -o "n=.*total.*" | sed "s/prep[^}]*tc_filter/tc_filter/; s/, .exact_knn.*}//; s/^/[cap=$cap] /"
  done
done
