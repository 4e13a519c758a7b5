for lib in build/libsor_k3d.so build/libsor_k3a.so build/libsor_k3b.so build/libsor_k3c.so; do
  SOR_LIBRARY=$lib timeout 600 python -m pytest tests/test_sor3d_gpu.py -q -m gpu -x 2>&1 | tail -2
  SOR_LIBRARY=$lib timeout 300 python tools/sor3d_perf.py
done > gpurun_out/r2_3d.log 2>&1
cat gpurun_out/r2_3d.log
