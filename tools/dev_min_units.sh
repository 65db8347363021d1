# Dev (GPU): CTA-count caps for small query sets (filter + re-rank per search)
for sh in "4800 4800 32" "2560 40000 64" "1024 100000 96" "9600 9600 96"; do
  for v in X=0 KNN_B200_CTAS_PER_PAIR=3 KNN_B200_CTAS_PER_PAIR=4 KNN_B200_CTAS_PER_PAIR=6 KNN_B200_CTAS_PER_PAIR=8; do
    env $v _FM_CHILD=1 timeout 60 python tools/filter_modes.py $sh 20 10 | sed "s/^/[$v] /"
  done
done
