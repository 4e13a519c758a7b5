"""One K7 launch per case for ncu (development aid): C2 iterate at T (argv[1],
default 3) on the multi-CTA form, C1 solve on the one-CTA form."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = SI.config("C2")
with P.Grid.create(torch.from_numpy(cfg.init()).cuda()) as g:
    g.set_kernel("resident", T)
    g.iterate(cfg.omega, cfg.iters)
c1 = SI.config("C1")
with P.Grid.create(torch.from_numpy(c1.init()).cuda()) as g:
    g.set_kernel("resident", 1)
    g.solve(c1.omega, c1.tol, c1.maxit, 1)
torch.cuda.synchronize()
