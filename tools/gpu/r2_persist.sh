timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -4 > gpurun_out/r2_persist_tests.log
for tps in 0 4 6 8; do SOR_PERSIST_TPS=$tps TAG=tps$tps python tools/c2_perf.py 1 2 3 4; done > gpurun_out/r2_c2.log 2>&1
SOR_NO_PERSIST=1 TAG=nopersist python tools/c2_perf.py 1 2 3 4 >> gpurun_out/r2_c2.log 2>&1
cat gpurun_out/r2_persist_tests.log gpurun_out/r2_c2.log
