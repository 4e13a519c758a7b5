"""K7 (SOR_KERNEL_RESIDENT) timing on the small BJ configs (development aid):
C2 (1024^2 f64, 2000 iterations) per-iteration time at T = 1..4 against the
wave kernels' best (temporal T=4 with K6), and C1 (64^2 solve, 1785 its) on
the one-CTA register form vs the shared-memory K5."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

cfg = SI.config("C2")
init = torch.from_numpy(cfg.init()).cuda()
for kernel, T in [("temporal", 4)] + [("resident", t) for t in (1, 2, 3, 4)]:
    for dtype in ("f64", "f32"):
        with P.Grid.create(init, dtype=dtype) as g:
            g.set_kernel(kernel, T)
            g.iterate(cfg.omega, 40)
            best = 1e30
            for _ in range(5):
                g.reset(init)
                g.iterate(cfg.omega, cfg.iters)
                best = min(best, g.elapsed_ms)
            st = g.stats
        print(f"C2 {kernel:9s} T={T} {dtype}: {best:8.3f} ms  {best * 1e3 / cfg.iters:6.3f} us/iter  "
              f"{cfg.rows * cfg.cols * cfg.iters / best / 1e6:7.1f} GLUP/s  launches={st['kernel_launches']}",
              flush=True)
c1 = SI.config("C1")
i1 = torch.from_numpy(c1.init()).cuda()
for kernel in ("small", "resident"):
    with P.Grid.create(i1) as g:
        g.set_kernel(kernel, 1)
        best = 1e30
        for _ in range(5):
            g.reset(i1)
            r = g.solve(c1.omega, c1.tol, c1.maxit, 1)
            best = min(best, g.elapsed_ms)
    print(f"C1 {kernel:9s}: {r.iters} its {best:8.3f} ms  {best * 1e3 / r.iters:6.3f} us/iter", flush=True)
