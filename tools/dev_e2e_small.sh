# Dev (GPU): host-API e2e vs pipeline chunk size on the smaller configs
E2E_SHAPE=19200,19200,96 E2E_CHUNKS=65536,9600,6400,4864 timeout 300 python tools/e2e_chunks.py
E2E_SHAPE=19200,19200,8 E2E_CHUNKS=65536,9600,6400 timeout 300 python tools/e2e_chunks.py
E2E_SHAPE=4800,4800,32 E2E_CHUNKS=65536,2560,1280 timeout 300 python tools/e2e_chunks.py
