"""3-D SOR (NEXT-3) throughput (development aid): 512^3 f64/f32, both kernels;
iterations 1-50 from the zero interior and 201-250 (the diffusion front then
carries many subnormal values through s/6's integer path)."""
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
            g.iterate(1.9, iters)
            t0 = g.elapsed_ms
            g.iterate(1.9, 150)
            g.iterate(1.9, iters)
            t1 = g.elapsed_ms
        esz = 8 if dtype == "f64" else 4
        bpu = (2 if kernel == "fused" else 4) * esz
        r0, r1 = n ** 3 * iters / t0 / 1e6, n ** 3 * iters / t1 / 1e6
        print(f"{os.path.basename(os.environ.get('SOR_LIBRARY', 'default')):8s} 3-D {n}^3 {kernel:8s} {dtype}: "
              f"its 1-50 {r0:6.1f} GLUP/s, its 201-250 {r1:6.1f} GLUP/s ({r1 * bpu:.0f} GB/s algorithmic at {bpu} B/update)",
              flush=True)
