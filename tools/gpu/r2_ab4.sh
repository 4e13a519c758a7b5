SOR_WAVE2=1 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -q -m gpu -x 2>&1 | tail -3
bash tools/ab.sh "C3:4 C3:4:solve C5:4 C3:3" paper_1401_0763_b200/libsor.so build/libsor_ring2.so build/libsor_ring4.so > gpurun_out/r2_ab4.log 2>&1
cat gpurun_out/r2_ab4.log
