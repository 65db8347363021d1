# Dev (GPU): large-k select over config D's k and other d (fallback counts + times)
bash tools/dev_sel_ab.sh
for sh in "38400 38400 128 1024" "38400 38400 8 256" "38400 38400 16 1024" "19200 19200 96 100"; do
  timeout 120 python tools/prof_shape.py $sh 2>&1 | tail -1 | sed 's/.prep_range[^}]*tc_filter_fixed/tc_filter_fixed/; s/, .exact_large_sample.*}//'
done
timeout 900 python -m pytest tests -m gpu -x -q -k "large or parity or select or certificate" 2>&1 | tail -2
