"""One C5 pass at depth T (argv[1]) for ncu (development aid)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402
T = int(sys.argv[1])
cfg = SI.config("C5")
with P.Grid.create(torch.from_numpy(cfg.init()).cuda()) as g:
    g.set_kernel("temporal", T)
    g.iterate(cfg.omega, 2 * T)
torch.cuda.synchronize()
