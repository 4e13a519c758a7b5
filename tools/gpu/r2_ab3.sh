bash tools/ab.sh "C3:4 C3:4:solve C5:4" paper_1401_0763_b200/libsor.so build/libsor_w2k4.so > gpurun_out/r2_ab3.log 2>&1
cat gpurun_out/r2_ab3.log
