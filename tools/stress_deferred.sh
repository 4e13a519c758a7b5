for env in "X=1" "SOR_NO_PDL=1" "SOR_NO_DEFER=1"; do
  for T in 3 4 2; do echo "== $env T=$T"; env $env timeout 200 python tools/stress_deferred.py $T 40 2>&1 | tail -4; done
done
