"""Replay one fuzz_solve case (development aid)."""
import random
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402


def replay(rows, cols, kernel, T, seed, ops, reps=5):
    init = SI.random_edges(rows, cols, seed=seed)
    bad = 0
    for rep in range(reps):
        ref = init.copy()
        with P.Grid.create(init) as g:
            g.set_kernel(kernel, T)
            for op in ops:
                if op[0] == "it":
                    g.iterate(op[1], op[2]); oracle.iterate(ref, op[1], op[2])
                elif op[0] == "reset":
                    g.reset(init); ref = init.copy()
                else:
                    _, omega, tol, maxit, K = op[:5]
                    r = g.solve(omega, tol, maxit, K)
                    rr = oracle.solve(ref, omega, tol, maxit, K)
                    if (r.iters, r.max_change) != (rr.iters, rr.max_change):
                        print("  solve mismatch", op[:5], r, rr.iters, rr.max_change)
                        bad += 1
            ok = np.array_equal(g.download(), ref)
            bad += not ok
    return bad


if __name__ == "__main__":
    ops = [("solve", 1.5, 0.0007223742349150175, 3000, 1), ("it", 1.5, 40), ("it", 1.5, 15),
           ("solve", 1.5, 3.922311077380035e-09, 37, 2)]
    print("full:", replay(228, 396, "temporal", 3, 548781, ops))
    print("no first solve:", replay(228, 396, "temporal", 3, 548781, ops[1:]))
    print("only last solve after 3055 its:", replay(228, 396, "temporal", 3, 548781, [("it", 1.5, 3000)] + ops[1:]))
    print("first solve + last:", replay(228, 396, "temporal", 3, 548781, [ops[0], ("it", 1.5, 55), ops[3]]))
