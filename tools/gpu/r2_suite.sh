timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 2>&1 | tail -30 > gpurun_out/r2_suite.log
SOR_NO_PERSIST=0 timeout 300 python tools/c2_perf.py 1 2 3 4 >> gpurun_out/r2_suite.log 2>&1
cat gpurun_out/r2_suite.log
