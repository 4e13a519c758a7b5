"""ncu driver for the NEXT rows (development aid): Jacobi C3 T=4 (8 passes) and 3-D 512^3 (3 iterations)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

which = sys.argv[1]
if which == "jacobi":
    cfg = SI.config("C3")
    with P.Grid.create(torch.from_numpy(cfg.init()).cuda()) as g:
        g.set_kernel("temporal", 4)
        g.jacobi(32)
        print(f"jacobi 32 its: {g.elapsed_ms:.3f} ms")
else:
    init = SI.random_shell3d(512, 512, 512, seed=7)
    with P.Grid3D(init) as g:
        g.iterate(1.9, 3)
        print(f"3d 3 its: {g.elapsed_ms:.3f} ms")
