"""C4 (16384^2, harmonic + noise boundary, omega 1.9, 500 iterations) at
temporal depth T, f64 and f32, device-timed (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

for name in ("C4",):
    cfg = SI.config(name)
    dinit = torch.from_numpy(cfg.init()).cuda()
    dtype = "f32" if name == "C4F32" else "f64"
    for T in (4, 5, 6):
        with P.Grid.create(dinit, dtype=dtype) as g:
            g.set_kernel("temporal", T)
            g.iterate(cfg.omega, 2 * T)
            best = 1e30
            for _ in range(3):
                g.reset(dinit)
                g.iterate(cfg.omega, cfg.iters)
                best = min(best, g.elapsed_ms)
        print(f"{name} {dtype} T={T}: {best:8.2f} ms  {cfg.rows * cfg.cols * cfg.iters / best / 1e6:7.1f} GLUP/s",
              flush=True)
