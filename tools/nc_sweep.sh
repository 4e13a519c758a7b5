# columns-per-lane sweep of the split wave kernel (development aid)
lib=$1
for nc in 4 6 8; do
  echo "NC=$nc"; SOR_WAVE_NC=$nc SOR_LIBRARY=$lib timeout 300 python tools/ab_perf.py C3:4 C3:3 C3:2 C5:4 C5:3 C3:4:solve C4F32:4
done
