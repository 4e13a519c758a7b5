timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_configs_gpu.py -q -m gpu -x -k "not paper_replay_full" 2>&1 | tail -2
bash tools/ab.sh "C3:4 C3:4:solve C5:4 C4:4 C3:2" paper_1401_0763_b200/libsor.so build/libsor_noskip.so 2>&1 | tail -10
for lib in paper_1401_0763_b200/libsor.so build/libsor_noskip.so; do
SOR_LIBRARY=$lib timeout 900 python bench.py --steps 10 --warmup 3 --no-c5 --cpu-window 2 > gpurun_out/r2_bench_skip.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_skip.log').read().strip().splitlines()[-1]); print('$lib', d['value'], d['fixed_phase_glups'], d['solve_phase_glups'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
done
