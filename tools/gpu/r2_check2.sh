set -x
timeout 1200 python -m pytest tests/test_configs_gpu.py -q -m gpu -k "multiwave or paper_replay_full" 2>&1 | tail -8 > gpurun_out/r2_cfg.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench2.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref.log 2>&1
timeout 600 python tools/cpu_gap_probe.py --cuda > gpurun_out/r2_gap.log 2>&1
timeout 600 python tools/cpu_gap_probe.py >> gpurun_out/r2_gap.log 2>&1
nproc >> gpurun_out/r2_gap.log; lscpu | head -20 >> gpurun_out/r2_gap.log
