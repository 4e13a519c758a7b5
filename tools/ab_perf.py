"""Best-of-N timing of a few (config, T, mode) points with the libsor named by
SOR_LIBRARY (development aid for A/B builds on one box).
usage: python tools/ab_perf.py C3:4 C5:4 C3:4:solve ..."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

tag = os.path.basename(os.environ.get("SOR_LIBRARY", "default"))
for spec in sys.argv[1:]:
    parts = spec.split(":")
    name, T = parts[0], int(parts[1])
    solve = len(parts) > 2 and parts[2] == "solve"
    dtype = "f32" if name.endswith("F32") else "f64"
    cfg = SI.config(name.replace("F32", ""), dtype=dtype)
    init = torch.from_numpy(cfg.init()).cuda()
    best = 1e30
    with P.Grid.create(init, dtype=dtype) as g:
        g.set_kernel("temporal" if T > 1 else "fused", T)
        for rep in range(3):
            g.reset(init)
            if solve:
                g.iterate(cfg.omega, cfg.iters)
                r = g.solve(cfg.omega, cfg.tol, cfg.maxit, cfg.check_every)
                n = r.iters
            else:
                n = cfg.iters
                g.iterate(cfg.omega, n)
            best = min(best, g.elapsed_ms)
    print(f"{tag:14s} {spec:12s} {n:6d} its {best:9.3f} ms {cfg.rows * cfg.cols * n / best / 1e6:8.1f} GLUP/s",
          flush=True)
