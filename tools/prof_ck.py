"""ncu driver: C3, T given, iterate 60 then solve(no conv) 60 with SOR_SOLVE_CK from env."""
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
    g.iterate(cfg.omega, 600)
    r = g.solve(cfg.omega, 1e-300, 60, 1)
    print(g.elapsed_ms, r)
