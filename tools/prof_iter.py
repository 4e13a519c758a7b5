"""ncu driver: C3 (or given config) fixed iterations with temporal depth T (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

cfgname, T, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = SI.config(cfgname)
init = torch.from_numpy(cfg.init()).cuda()
with P.Grid.create(init) as g:
    g.set_kernel("temporal", T)
    g.iterate(cfg.omega, iters)
    print(f"{cfgname} T={T} {iters} iters: {g.elapsed_ms:.3f} ms, {cfg.rows * cfg.cols * iters / g.elapsed_ms / 1e6:.1f} GLUP/s")
