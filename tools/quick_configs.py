"""Throughput survey of the other BASELINE configs (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402


def run(name, dtype, kernel, T, iters=None, solve=False):
    cfg = SI.config(name, dtype=dtype)
    init = torch.from_numpy(cfg.init()).cuda()
    with P.Grid.create(init, dtype=dtype) as g:
        g.set_kernel(kernel, T)
        if solve:
            g.solve(cfg.omega, cfg.tol, cfg.maxit, cfg.check_every)
            g.reset(init)
            r = g.solve(cfg.omega, cfg.tol, cfg.maxit, cfg.check_every)
            n = r.iters
        else:
            n = iters or cfg.iters
            g.iterate(cfg.omega, min(n, 50))
            g.reset(init)
            g.iterate(cfg.omega, n)
        ms = g.elapsed_ms
    print(f"{name} {dtype} {kernel:8s} T={T}: {n} its {ms:9.3f} ms {cfg.rows*cfg.cols*n/ms/1e6:8.1f} GLUP/s "
          f"({ms*1e3/n:.2f} us/iter)", flush=True)


for k, T in (("small", 1), ("fused", 1), ("temporal", 2), ("temporal", 4), ("natural", 1)):
    run("C1", "f64", k, T, solve=True)
for k, T in (("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4)):
    run("C2", "f64", k, T)
for dt in ("f64", "f32"):
    for k, T in (("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4)):
        run("C4", dt, k, T)
