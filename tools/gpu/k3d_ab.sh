for i in 1 2; do python tools/sor3d_perf.py 2>&1 | grep fused; SOR_LIBRARY=paper_1401_0763_b200/libsor_tinycall.so python tools/sor3d_perf.py 2>&1 | grep fused; done
