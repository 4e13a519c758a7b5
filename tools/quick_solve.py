"""C3 solve-phase timing per kernel variant (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

cfg = SI.config(sys.argv[1] if len(sys.argv) > 1 else "C3")
init = torch.from_numpy(cfg.init()).cuda()
for kernel, T in (("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4)):
    with P.Grid.create(init) as g:
        g.set_kernel(kernel, T)
        g.iterate(cfg.omega, cfg.iters)
        t_it = g.elapsed_ms
        r = g.solve(cfg.omega, cfg.tol, cfg.maxit, cfg.check_every)
        t_s = g.elapsed_ms
        st = g.stats
        print(f"{kernel:9s} T={T}: iterate {cfg.iters} in {t_it:8.2f} ms ({cfg.rows*cfg.cols*cfg.iters/t_it/1e6:7.1f} GLUP/s); "
              f"solve {r.iters} its conv={r.converged} max={r.max_change:.4e} in {t_s:8.2f} ms "
              f"({cfg.rows*cfg.cols*r.iters/t_s/1e6:7.1f} GLUP/s) launches={st['kernel_launches']} reruns={st['exact_reruns']}", flush=True)
