"""Cost of the solve-mode max-change (ck=3/4) vs plain passes, C3, no convergence."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

cfg = SI.config("C3")
init = torch.from_numpy(cfg.init()).cuda()
for T in (2, 3, 4):
    with P.Grid.create(init) as g:
        g.set_kernel("temporal", T)
        g.iterate(cfg.omega, 120)
        g.reset(init)
        g.iterate(cfg.omega, 1200)
        t_it = g.elapsed_ms
        g.reset(init)
        r = g.solve(cfg.omega, 1e-300, 1200, 1)
        t_sv = g.elapsed_ms
        print(f"T={T} ck={os.environ.get('SOR_SOLVE_CK', 'auto')}: iterate {t_it:.2f} ms, solve(no conv) {t_sv:.2f} ms "
              f"ratio {t_sv / t_it:.3f} launches {g.stats['kernel_launches']}", flush=True)
