timeout 600 python -m pytest tests/test_sor3d_gpu.py tests/test_bench_contract.py -q -m gpu -x -k "sor3d" 2>&1 | tail -2
timeout 300 python tools/sor3d_perf.py
SOR_3D_NOSPLIT=1 timeout 300 python tools/sor3d_perf.py | grep natural
