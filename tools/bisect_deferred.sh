for env in "X=1" "SOR_NO_PDL=1" "SOR_NO_DEFER=1" "SOR_NO_PDL=1 SOR_NO_DEFER=1"; do
  echo "== $env"
  env $env timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "deferred" 2>&1 | tail -3
done
