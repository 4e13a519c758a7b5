# rerun the GPU parity suite several times per environment to catch a flaky failure (development aid)
for env in "X=1" "SOR_NO_PDL=1"; do
  for i in 1 2 3 4; do
    env $env timeout 300 python -m pytest tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/flaky.log 2>&1
    echo "== $env run $i: $(tail -n 1 gpurun_out/flaky.log)"
    grep -h "^E  \|FAILED" gpurun_out/flaky.log | head -8
  done
done
