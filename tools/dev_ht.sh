# Dev (GPU): host-side timing of one tensor search (variant build with HT checkpoints)
KNN_HT=1 _KNN_B200_DEV_LIB=build_variants/ht3/libknn_b200.so timeout 120 python tools/oneshot_wall.py 2>&1 | head -60
