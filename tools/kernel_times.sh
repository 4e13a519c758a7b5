# ncu launch list of a short C3 solve for several libsor builds (development aid):
#   tools/kernel_times.sh lib1 lib2 ...   -> gpurun_out/kt_<lib>.csv
for lib in "$@"; do
  b=$(basename $lib .so)
  SOR_LIBRARY=$lib python tools/prof_solve.py 4 > gpurun_out/kt_$b.log 2>&1 &&
  SOR_LIBRARY=$lib ncu --metrics gpu__time_duration.sum --clock-control none -s 240 -c 60 --csv \
      --log-file gpurun_out/kt_$b.csv python tools/prof_solve.py 4 > /dev/null 2>&1
done
