# Round-2 measurements of the new kernels: headline bench (with the C1/C2 sub-record), the NEXT-3
# line, ncu captures of the K7 (C2) and k3d_tma launches
python bench.py > gpurun_out/r2_bench_k7.json 2> gpurun_out/r2_bench_k7.err
python bench.py --method sor3d --steps 3 --warmup 3 > gpurun_out/r2_bench_next3_tma.json 2> gpurun_out/r2_bench_next3_tma.err
ncu --set full --import-source on --clock-control none -k regex:resident_kernel -c 2 -o gpurun_out/r2_ncu_k7 python tools/prof_k7.py 3 > gpurun_out/r2_ncu_k7.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k3d_tma -s 1 -c 1 -o gpurun_out/r2_ncu_k3d_tma python tools/prof_3d.py > gpurun_out/r2_ncu_k3d.log 2>&1
tail -c 600 gpurun_out/r2_bench_k7.json
