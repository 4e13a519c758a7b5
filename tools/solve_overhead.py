"""Per-pass cost of the solve loop vs plain iteration on C3, T=4 (development aid):
iterate(3000) vs solve(tol=1e-300, maxit=3000, K=1) (never converges: every pass a probe pass)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

cfg = SI.config("C3")
init = torch.from_numpy(cfg.init()).cuda()
with P.Grid.create(init) as g:
    g.set_kernel("temporal", 4)
    g.iterate(cfg.omega, 100)
    for rep in range(2):
        g.reset(init)
        g.iterate(cfg.omega, 3000)
        ti = g.elapsed_ms
        g.reset(init)
        r = g.solve(cfg.omega, 1e-300, 3000, 1)
        ts = g.elapsed_ms
        st = g.stats
        print(f"iterate 3000: {ti:.2f} ms ({ti * 1e3 / 750:.2f} us/pass); solve 3000 (no convergence): {ts:.2f} ms "
              f"({ts * 1e3 / 750:.2f} us/pass) launches={st['kernel_launches']} reruns={st['exact_reruns']}", flush=True)
