SOR_WAVE2_NWT=4 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_configs_gpu.py -q -m gpu -x -k "not paper_replay_full" 2>&1 | tail -3
for v in 2 4 2 4; do SOR_WAVE2_NWT=$v timeout 300 python tools/ab_perf.py C3:4 C3:4:solve C5:4 C4:4 | sed "s/^/nwt=$v /"; done
