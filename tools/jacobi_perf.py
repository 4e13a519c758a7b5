"""Jacobi (NEXT-2) throughput survey (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

for name, iters in (("C3", 1000), ("C5", 200)):
    cfg = SI.config(name)
    init = torch.from_numpy(cfg.init()).cuda()
    for kernel, T in (("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4)):
        with P.Grid.create(init) as g:
            g.set_kernel(kernel, T)
            g.jacobi(min(iters, 40))
            best = 1e30
            for _ in range(2):
                g.reset(init)
                g.jacobi(iters)
                best = min(best, g.elapsed_ms)
        glups = cfg.rows * cfg.cols * iters / best / 1e6
        print(f"Jacobi {name} {kernel:8s} T={T}: {iters} its {best:9.3f} ms {glups:8.1f} GLUP/s "
              f"({glups * 16 / T:.0f} GB/s algorithmic)", flush=True)
