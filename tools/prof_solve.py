"""ncu driver: C3 iterate(1000) then a short solve (ck=2 passes) with the given T."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

T = int(sys.argv[1])
cfg = SI.config("C3")
init = torch.from_numpy(cfg.init()).cuda()
with P.Grid.create(init) as g:
    g.set_kernel("temporal", T)
    g.iterate(cfg.omega, 1000)
    r = g.solve(cfg.omega, cfg.tol, 96, 1)
    print(f"T={T} solve 96: {g.elapsed_ms:.3f} ms, {r}")
