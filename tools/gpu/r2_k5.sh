timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -q -m gpu -x -k "small or c1" 2>&1 | tail -3
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_1401_0763_b200 as P, sor_inputs as SI
cfg = SI.config("C1")
for kernel, T in (("small", 1), ("temporal", 3), ("temporal", 4), ("fused", 1)):
    best = 1e9
    with P.Grid.create(cfg.init()) as g:
        g.set_kernel(kernel, T)
        for _ in range(5):
            g.reset(cfg.init())
            r = g.solve(cfg.omega, cfg.tol, cfg.maxit, 1)
            best = min(best, g.elapsed_ms)
    print(f"C1 {kernel} T={T}: {r.iters} its {best:.3f} ms {best * 1e3 / r.iters:.3f} us/iter", flush=True)
PY
