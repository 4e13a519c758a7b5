# solve polling batch sweep (development aid)
for b in 32 64 128 256 512; do echo -n "batch=$b "; SOR_SOLVE_BATCH=$b SOR_LIBRARY=build/libsor_B.so python tools/ab_perf.py C3:4:solve | sed -E 's/ +[0-9]+ its//' ; done
