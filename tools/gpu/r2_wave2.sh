export SOR_WAVE2=1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -x 2>&1 | tail -5 > gpurun_out/r2_w2_tests.log
timeout 900 python -m pytest tests/test_fuzz_gpu.py tests/test_configs_gpu.py -q -m gpu -x -k "not paper_replay_full" 2>&1 | tail -5 >> gpurun_out/r2_w2_tests.log
cat gpurun_out/r2_w2_tests.log
for v in 0 1 0 1; do SOR_WAVE2=$v timeout 300 python tools/ab_perf.py C3:4 C3:4:solve C5:4 C3:3 C3:2 | sed "s/^/w2=$v /"; done > gpurun_out/r2_w2_perf.log 2>&1
cat gpurun_out/r2_w2_perf.log
