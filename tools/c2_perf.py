"""C2 (1024^2 f64, 2000 iterations, L2-resident) per-iteration time for the
kernel paths (development aid): python tools/c2_perf.py [T ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

cfg = SI.config("C2")
init = torch.from_numpy(cfg.init()).cuda()
tag = os.environ.get("TAG", "")
for T in [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4]:
    with P.Grid.create(init) as g:
        g.set_kernel("temporal" if T > 1 else "fused", T)
        g.iterate(cfg.omega, 40)
        best = 1e30
        for _ in range(5):
            g.reset(init)
            g.iterate(cfg.omega, cfg.iters)
            best = min(best, g.elapsed_ms)
        st = g.stats
    print(f"{tag:10s} C2 T={T}: {best:8.3f} ms  {best * 1e3 / cfg.iters:6.3f} us/iter  "
          f"{cfg.rows * cfg.cols * cfg.iters / best / 1e6:7.1f} GLUP/s  launches={st['kernel_launches']}", flush=True)
