# NEXT-3 one-pass TMA kernel: tests, then 512^3 throughput (both kernels), ncu of the fused kernel
timeout 600 python -m pytest tests/test_sor3d_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
python tools/sor3d_perf.py
SOR_K3T_F32=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import paper_1401_0763_b200 as P, sor_inputs as SI
init = SI.random_shell3d(4, 5, 6, seed=1)
with P.Grid3D(init, dtype='f32') as g:
    g.set_kernel('fused'); g.iterate(1.5, 2); print('f32 tma ok')
" 2>&1 | tail -2
ncu --set full --import-source on --clock-control none -k regex:k3d_tma -s 1 -c 1 -o gpurun_out/k3d_h python tools/prof_3d.py > /dev/null 2>&1
