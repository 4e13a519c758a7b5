"""Quick GLUP/s survey of the kernel variants (development aid, not the bench contract)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402


def run(cfgname, kernel, T, iters, dtype="f64", reps=3):
    cfg = SI.config(cfgname, dtype=dtype)
    init = torch.from_numpy(cfg.init()).cuda()
    g = P.Grid.create(init, dtype=dtype)
    g.set_kernel(kernel, T)
    g.iterate(cfg.omega, min(iters, 20))
    best = 1e30
    for _ in range(reps):
        g.reset(init)
        g.iterate(cfg.omega, iters)
        best = min(best, g.elapsed_ms)
    st = g.stats
    g.close()
    glups = cfg.rows * cfg.cols * iters / (best * 1e-3) / 1e9
    esz = 8 if dtype == "f64" else 4
    gbs = glups * 2 * esz
    print(f"{cfgname} {dtype} {kernel:9s} T={T} iters={iters}: {best:9.3f} ms  {glups:8.1f} GLUP/s  "
          f"alg {gbs:7.0f} GB/s/pass-equiv  launches={st['kernel_launches']}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["C3"]
    for c in which:
        iters = {"C2": 2000, "C3": 1000, "C4": 500, "C5": 200}[c]
        for dtype in (["f64", "f32"] if c == "C4" else ["f64"]):
            for k, T in (("natural", 1), ("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4)):
                run(c, k, T, iters, dtype)
