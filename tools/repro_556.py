"""Replay fuzz case (seed 21, case 556) many times against one oracle run
(development aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

rows, cols, kernel, T, seed = 379, 540, "temporal", 2, 783207
ops = [("it", 1.0, 38), ("it", 1.97, 32), ("it", 1.9, 40), ("solve", 0.376, 7.069788613454461e-09, 3000, 1),
       ("solve", 1.97, 1.0129908223994698e-07, 3000, 5)]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
init = SI.random_edges(rows, cols, seed=seed)
ref = init.copy()
want = []
for op in ops:
    if op[0] == "it":
        oracle.iterate(ref, op[1], op[2])
    else:
        rr = oracle.solve(ref, *op[1:5]); want.append((rr.iters, rr.max_change))
bad = 0
for rep in range(reps):
    with P.Grid.create(init) as g:
        g.set_kernel(kernel, T)
        got = []
        for op in ops:
            if op[0] == "it":
                g.iterate(op[1], op[2])
            else:
                r = g.solve(*op[1:5]); got.append((r.iters, r.max_change))
        ok = got == want and np.array_equal(g.download(), ref)
        if not ok:
            bad += 1
            print("bad rep", rep, got, want, flush=True)
print(f"{reps} reps, {bad} bad")
