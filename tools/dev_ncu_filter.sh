# ncu --set full of the small-k filter on config B (dev): $1 = output name, rest = env assignments
out=$1; shift
env "$@" _FM_CHILD=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"filter" -s 1 -c 1 -o gpurun_out/$out -f python tools/filter_modes.py 38400 38400 96 20 2 > gpurun_out/$out.log 2>&1
