timeout 900 python -m pytest tests/test_bench_contract.py -q -m gpu -x 2>&1 | tail -4 > gpurun_out/r2_2rank.log
cat gpurun_out/r2_2rank.log
python tools/prof_iter.py C3 4 40 > gpurun_out/r3_plain_it.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:wave2_kernel -s 6 -c 1 -o gpurun_out/r3_c3_it_T4 python tools/prof_iter.py C3 4 40 > gpurun_out/r3_ncu_it.log 2>&1
python tools/prof_solve.py 4 > gpurun_out/r3_plain_solve.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:wave2_kernel -s 262 -c 1 -o gpurun_out/r3_c3_solve_T4 python tools/prof_solve.py 4 > gpurun_out/r3_ncu_solve.log 2>&1
python tools/prof_iter.py C5 4 40 > gpurun_out/r3_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:wave2_kernel -s 6 -c 1 -o gpurun_out/r3_c5_T4 python tools/prof_iter.py C5 4 40 > gpurun_out/r3_ncu_c5.log 2>&1
python bench.py --steps 1 --warmup 3 --no-c5 --no-e2e --cpu-window 2 > gpurun_out/r3_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r3_launches.csv python bench.py --steps 1 --warmup 3 --no-c5 --no-e2e --cpu-window 2 > gpurun_out/r3_ncu_bench.log 2>&1
ls -la gpurun_out/ | grep r3_
