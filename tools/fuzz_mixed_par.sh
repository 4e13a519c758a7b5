# N parallel mixed SOR/Jacobi fuzzers sharing the GPU (development aid)
S=${1:-480}; N=${2:-8}; B=${3:-200}
for i in $(seq 0 $((N - 1))); do
  python tools/fuzz_mixed.py "$S" $((B + i)) > gpurun_out/fzm_$((B + i)).log 2>&1 &
done
wait
grep -h "MISMATCH\|fuzz-mixed:" gpurun_out/fzm_*.log
