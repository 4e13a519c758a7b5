"""Small driver for ncu captures: one config, one kernel variant, a few passes."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

cfgname, kernel, T, iters = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
dtype = sys.argv[5] if len(sys.argv) > 5 else "f64"
cfg = SI.config(cfgname, dtype=dtype)
init = torch.from_numpy(cfg.init()).cuda()
with P.Grid.create(init, dtype=dtype) as g:
    g.set_kernel(kernel, T)
    g.iterate(cfg.omega, iters)
    print(f"{cfgname} {kernel} T={T} {iters} iters: {g.elapsed_ms:.3f} ms, "
          f"{cfg.rows * cfg.cols * iters / g.elapsed_ms / 1e6:.1f} GLUP/s, stats {g.stats}")
