# N parallel fuzzers sharing the GPU (development aid): bash tools/fuzz_par.sh SECONDS N SEED0
S=${1:-600}; N=${2:-8}; B=${3:-100}
for i in $(seq 0 $((N - 1))); do
  python tools/fuzz_solve.py "$S" $((B + i)) > gpurun_out/fzp_$((B + i)).log 2>&1 &
done
wait
grep -h "MISMATCH\|fuzz:" gpurun_out/fzp_*.log
