SOR_RES_VERBOSE=1 SOR_RES_RPW=2 SOR_RESIDENT_T=1 python tools/k7_perf.py 2>&1 | head -3
for b in 0 100 400; do SOR_RES_BACKOFF=$b RPWS=4 TS="1 3" bash tools/gpu/k7ab.sh; done
python tools/k7_trace.py
