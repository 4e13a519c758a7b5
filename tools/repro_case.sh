for env in "X=1" "SOR_NO_PDL=1" "SOR_NO_DEFER=1" "SOR_NO_PDL=1 SOR_NO_DEFER=1"; do echo "== $env"; env $env timeout 120 python tools/repro_case.py; done
