timeout 900 python -m pytest tests/test_dist_gpu.py -q -m gpu -x 2>&1 | tail -2
for s in 1 2 3; do timeout 1500 python tools/fuzz_dist_ipc.py launch $((s + 1)) 500 $((800 + s)); done 2>&1 | grep -E "fuzz_dist|MISMATCH|Error|error" | tee gpurun_out/r2_dfuzz2.txt
