"""C5 (32768^2 f64, omega_opt, 200 iterations) at temporal depth T (argv),
device-timed (development aid; the bench's c5 sub-record runs T = 4)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

cfg = SI.config("C5")
dinit = torch.from_numpy(cfg.init()).cuda()
for T in [int(x) for x in sys.argv[1:]] or [4, 5, 6]:
    with P.Grid.create(dinit) as g:
        g.set_kernel("temporal", T)
        g.iterate(cfg.omega, 2 * T)
        ms = []
        for _ in range(3):
            g.reset(dinit)
            g.iterate(cfg.omega, cfg.iters)
            ms.append(g.elapsed_ms)
    best = min(ms)
    print(f"C5 T={T}: {best:8.2f} ms  {cfg.rows * cfg.cols * cfg.iters / best / 1e6:7.1f} GLUP/s", flush=True)
    del g
