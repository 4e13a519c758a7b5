# alpha sweep of the one-wave tiling (development aid): tools/alpha_sweep.sh "1.15 1.33" "1.15 1.3 1.5"
for al in $1; do for a2 in $2; do echo -n "alpha=$al alpha2=$a2 "; SOR_WAVE_ALPHA=$al SOR_WAVE_ALPHA2=$a2 python tools/ab_perf.py C3:4 C3:3 C2:4 | sed -E 's/ +[0-9]+ its +[0-9.]+ ms//; s/default +//' | tr '\n' ' '; echo; done; done
