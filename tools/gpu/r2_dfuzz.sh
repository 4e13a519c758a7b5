timeout 900 python -m pytest tests/test_dist_gpu.py -q -m gpu -x -k random 2>&1 | tail -3
for s in 1 2 3; do timeout 1200 python tools/fuzz_dist_ipc.py launch $((s + 1)) 60 $((700 + s)); done 2>&1 | grep -E "fuzz_dist|MISMATCH|Error|error" | tee gpurun_out/r2_dfuzz.txt
