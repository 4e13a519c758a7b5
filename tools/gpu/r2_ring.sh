timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_configs_gpu.py -q -m gpu -x -k "not paper_replay_full" 2>&1 | tail -3
for v in 1 2; do timeout 300 python tools/ab_perf.py C3:4 C3:4:solve C5:4 C3:3 C4:4; done
bash tools/gpu/r2_fuzz.sh 480
