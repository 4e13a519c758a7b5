for i in 0 1 2 3; do SOR_NO_PDL=1 python tools/fuzz_solve.py 420 $((400 + i)) > gpurun_out/fzf_nopdl_$i.log 2>&1 & done
for i in 0 1 2 3; do SOR_NO_DEFER=1 python tools/fuzz_solve.py 420 $((500 + i)) > gpurun_out/fzf_nodefer_$i.log 2>&1 & done
wait; grep -H "MISMATCH\|fuzz:" gpurun_out/fzf_*.log
