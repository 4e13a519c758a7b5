# PDL on/off A/B (development aid)
for rep in 1 2; do
  SOR_NO_PDL=1 SOR_LIBRARY=build/libsor_D3.so timeout 200 python tools/ab_perf.py C3:4 C3:4:solve C5:4 C3:1 | sed 's/^/nopdl /'
  SOR_LIBRARY=build/libsor_D3.so timeout 200 python tools/ab_perf.py C3:4 C3:4:solve C5:4 C3:1 | sed 's/^/pdl   /'
done
