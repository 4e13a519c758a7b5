timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -2
TAG=w2persist timeout 300 python tools/c2_perf.py 2 3 4
SOR_WAVE2=0 TAG=w1persist timeout 300 python tools/c2_perf.py 2 3 4
SOR_NO_PERSIST=1 TAG=w2launch timeout 300 python tools/c2_perf.py 2 3 4
SOR_PERSIST_TPS=8 TAG=w2p_tps8 timeout 300 python tools/c2_perf.py 2 3 4
SOR_PERSIST_TPS=3 TAG=w2p_tps3 timeout 300 python tools/c2_perf.py 2 3 4
SOR_PERSIST_TPS=2 TAG=w2p_tps2 timeout 300 python tools/c2_perf.py 2 3 4
