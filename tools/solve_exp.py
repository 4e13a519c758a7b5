"""Solve-phase experiment (development aid): python tools/solve_exp.py CFG T [pre_iters]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

name, T = sys.argv[1], int(sys.argv[2])
cfg = SI.config(name)
pre = int(sys.argv[3]) if len(sys.argv) > 3 else (cfg.iters or 0)
init = torch.from_numpy(cfg.init()).cuda()
tol = cfg.tol or 1e-8
maxit = cfg.maxit or 200000
with P.Grid.create(init) as g:
    g.set_kernel("temporal" if T > 1 else "fused", T)
    for rep in range(2):
        g.reset(init)
        if pre:
            g.iterate(cfg.omega, pre)
        r = g.solve(cfg.omega, tol, maxit, 1)
        st = g.stats
        print(f"{name} T={T}: {r.iters} its conv={r.converged} max={r.max_change:.6e} {g.elapsed_ms:.2f} ms "
              f"{cfg.rows * cfg.cols * r.iters / g.elapsed_ms / 1e6:.1f} GLUP/s reruns={st['exact_reruns']} "
              f"launches={st['kernel_launches']}", flush=True)
