for env in "X=1" "SOR_NO_PDL=1"; do echo "== $env"; env $env timeout 400 python tools/repro_556.py 150; done
