# NEXT-3 two-row kernel: fuzz (K7 + 3-D), NEXT-3 bench line, ncu capture of the f64 kernel
python tools/fuzz_k7.py 300 3 > gpurun_out/fuzz_k7_b.txt 2>&1
python bench.py --method sor3d --steps 3 --warmup 3 > gpurun_out/r2_bench_next3_tma2.json 2> gpurun_out/r2_bench_next3_tma2.err
ncu --set full --import-source on --clock-control none -k regex:k3d_tma -s 1 -c 1 -o gpurun_out/r2_ncu_k3d_tma2 python tools/prof_3d.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k3d_tma -s 1 -c 1 -o gpurun_out/r2_ncu_k3d_tma2_f32 python tools/prof_3d.py f32 > /dev/null 2>&1
cat gpurun_out/fuzz_k7_b.txt
