set -x
bash tools/ab.sh "C3:4 C3:4:solve C5:4" build/libsor_mix0.so build/libsor_mix1.so build/libsor_k4.so build/libsor_hoist.so > gpurun_out/r2_ab1.log 2>&1
cat gpurun_out/r2_ab1.log | tail -30
