S=${1:-600}
for i in $(seq 0 11); do
  timeout $((S + 300)) python tools/fuzz_r2.py "$S" $((500 + i)) > gpurun_out/fz2_$((500 + i)).log 2>&1 &
done
wait
grep -h "MISMATCH\|fuzz_r2" gpurun_out/fz2_*.log | tee gpurun_out/r2_fuzz_summary.txt
