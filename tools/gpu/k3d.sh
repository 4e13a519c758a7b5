# NEXT-3 one-pass TMA kernel: tests, then 512^3 throughput (both kernels)
timeout 600 python -m pytest tests/test_sor3d_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
python tools/sor3d_perf.py
