# alpha sweep of the one-wave tiling (development aid): tools/alpha_sweep.sh lib "1.2 1.33 1.5" "1.55"
lib=$1
for al in $2; do for a2 in $3; do echo -n "alpha=$al alpha2=$a2 "; SOR_WAVE_ALPHA=$al SOR_WAVE_ALPHA2=$a2 SOR_LIBRARY=$lib python tools/ab_perf.py C3:4 C3:3 C3:2 | sed -E 's/ +[0-9]+ its +[0-9.]+ ms//' | tr '\n' ' '; echo; done; done
