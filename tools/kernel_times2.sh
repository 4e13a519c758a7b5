# ncu launch list of a C3 solve (fixed maxit, no convergence) for several libsor builds (development aid)
for lib in "$@"; do
  b=$(basename $lib .so)
  SOR_LIBRARY=$lib timeout 120 python tools/prof_solve.py 4 > gpurun_out/kt2_$b.log 2>&1 &&
  SOR_LIBRARY=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 240 -c 40 --csv \
      --log-file gpurun_out/kt2_$b.csv python tools/prof_solve.py 4 > /dev/null 2>&1
done
