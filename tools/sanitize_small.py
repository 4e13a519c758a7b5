"""Small end-to-end run for compute-sanitizer (development aid): every kernel
variant on small grids, iterate + solve, f64 and f32, single and virtual slabs."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

for dtype in ("f64", "f32"):
    for kernel, T in (("natural", 1), ("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4), ("small", 1)):
        init = SI.random_edges(67, 150, seed=3)
        ref = oracle.to_storage(init, dtype)
        oracle.iterate(ref, 1.8, 9)
        with P.Grid.create(init, dtype=dtype) as g:
            g.set_kernel(kernel, T)
            g.iterate(1.8, 9)
            assert np.array_equal(g.download(), ref.astype(np.float64)), (dtype, kernel, T)
            g.solve(1.8, 1e-6, 400, 1)
        if kernel != "small":
            with P.Grid.create_virtual(init, 3, dtype=dtype) as g:
                g.set_kernel(kernel, T)
                g.iterate(1.8, 9)
                g.solve(1.8, 1e-6, 200, 2)
print("sanitize run ok")
