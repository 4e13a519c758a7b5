"""3-D SOR (NEXT-3) throughput (development aid): 512^3 f64/f32, fixed iterations, both kernels."""
import os
import sys

sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

n, iters = 512, 50
init = SI.random_shell3d(n, n, n, seed=7)
for kernel in ("fused", "natural"):
    for dtype in ("f64", "f32"):
        with P.Grid3D(init, dtype=dtype) as g:
            g.set_kernel(kernel)
            g.iterate(1.9, 5)
            best = min((g.iterate(1.9, iters), g.elapsed_ms)[1] for _ in range(3))
        glups = n ** 3 * iters / best / 1e6
        esz = 8 if dtype == "f64" else 4
        bpu = (2 if kernel == "fused" else 4) * esz
        print(f"{os.path.basename(os.environ.get('SOR_LIBRARY', 'default')):14s} 3-D {n}^3 {kernel:8s} {dtype}: {iters} its {best:8.2f} ms {glups:7.1f} GLUP/s "
              f"({glups * bpu:.0f} GB/s algorithmic at {bpu} B/update)", flush=True)
