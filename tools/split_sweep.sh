for sp in 1 0; do echo "split=$sp"; SOR_WAVE_SPLIT=$sp SOR_LIBRARY=build/libsor_I.so python tools/ab_perf.py C3:2 C3:3 C3:4 C5:3 C5:4; done
