timeout 1500 python -m pytest tests -q -m gpu -x -k "not paper_replay_full" 2>&1 | tail -4 > gpurun_out/r2_w2b_tests.log
SOR_WAVE2=0 SOR_NO_PERSIST=1 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -q -m gpu -x 2>&1 | tail -3 >> gpurun_out/r2_w2b_tests.log
cat gpurun_out/r2_w2b_tests.log
for v in 0 1 0 1; do SOR_WAVE2=$v timeout 300 python tools/ab_perf.py C3:4 C3:4:solve C5:4 | sed "s/^/w2=$v /"; done > gpurun_out/r2_w2b_perf.log 2>&1
cat gpurun_out/r2_w2b_perf.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench3.log 2>&1
tail -c 3000 gpurun_out/r2_bench3.log
