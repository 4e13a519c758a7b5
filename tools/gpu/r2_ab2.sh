bash tools/ab.sh "C3:4 C3:4:solve C5:4" build/libsor_mix0.so build/libsor_k4b.so build/libsor_hoistb.so build/libsor_k4h.so > gpurun_out/r2_ab2.log 2>&1
cat gpurun_out/r2_ab2.log | tail -24
