timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -q -m gpu -x 2>&1 | tail -2
for v in 1 2; do timeout 300 python tools/ab_perf.py C3:4 C3:4:solve; done
timeout 900 python bench.py --steps 10 --warmup 3 --no-c5 > gpurun_out/r2_bench5.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench5.log').read().strip().splitlines()[-1]); print(d['value'], d['fixed_phase_glups'], d['solve_phase_glups'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
