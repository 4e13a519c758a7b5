"""ncu driver for the NEXT-4 multi-colour kernel (development aid): 3 iterations on the C3 grid.
usage: python tools/prof_mc.py ca,cb,nc"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

ca, cb, nc = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,1,4").split(","))
cfg = SI.config("C3")
with P.Grid.create(torch.from_numpy(cfg.init()).cuda()) as g:
    g.variant_iterate(P.Variant.multicolor(ca, cb, nc), cfg.omega, 3)
    print(f"mc ({ca},{cb},{nc}) 3 its: {g.elapsed_ms:.3f} ms")
