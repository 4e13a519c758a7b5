timeout 1800 python -m pytest tests -q -m gpu -x --durations=8 2>&1 | tail -16 > gpurun_out/r2_final_suite.log
cat gpurun_out/r2_final_suite.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_final_bench.log 2>&1
tail -c 2500 gpurun_out/r2_final_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_final_ref.log 2>&1
tail -c 800 gpurun_out/r2_final_ref.log
