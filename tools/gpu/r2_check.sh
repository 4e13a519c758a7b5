set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/r2_dist.log
timeout 900 python -m pytest tests -q -m gpu -x --deselect tests/test_dist_gpu.py 2>&1 | tail -30 > gpurun_out/r2_all.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.log 2>&1
tail -3 gpurun_out/r2_dist.log gpurun_out/r2_all.log gpurun_out/r2_bench.log
