"""Stress the deferred solve (development aid): repeated solves on one handle vs the oracle."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

T = int(sys.argv[1])
reps = int(sys.argv[2])
init = SI.random_edges(300, 517, seed=40 + T)
ref = init.copy()
rr = oracle.solve(ref, 1.95, 1e-7, 20000, 1)
ref2 = ref.copy()
oracle.iterate(ref2, 1.95, 7)
rr2 = oracle.solve(ref2, 1.95, 1e-9, 20000, 1)
bad = 0
with P.Grid.create(init) as g:
    g.set_kernel("temporal" if T > 1 else "fused", T)
    for i in range(reps):
        g.reset(init)
        r = g.solve(1.95, 1e-7, 20000, 1)
        ok1 = (r.iters, r.max_change) == (rr.iters, rr.max_change) and np.array_equal(g.download(), ref)
        g.iterate(1.95, 7)
        r2 = g.solve(1.95, 1e-9, 20000, 1)
        ok2 = (r2.iters, r2.max_change) == (rr2.iters, rr2.max_change) and np.array_equal(g.download(), ref2)
        if not (ok1 and ok2):
            bad += 1
            print(f"rep {i}: first {r.iters}/{rr.iters} ok={ok1}; second {r2.iters}/{rr2.iters} ok={ok2} "
                  f"reruns={g.stats['exact_reruns']}", flush=True)
print(f"T={T}: {bad} bad of {reps}")
