"""Randomised differential test of interleaved SOR / Jacobi (NEXT-2) calls on
one handle against the oracle (development aid).
usage: python tools/fuzz_mixed.py SECONDS [seed]"""
import random
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

budget = float(sys.argv[1])
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
t0 = time.time()
n = bad = 0
while time.time() - t0 < budget:
    rows, cols = rng.randint(1, 400), rng.randint(1, 700)
    kernel, T = rng.choice([("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4)])
    dtype = rng.choice(["f64", "f64", "f32"])
    init = SI.random_edges(rows, cols, seed=rng.randint(0, 10**6))
    ref = oracle.to_storage(init, dtype)
    log = []
    with P.Grid.create(init, dtype=dtype) as g:
        g.set_kernel(kernel, T)
        for _ in range(rng.randint(2, 6)):
            op = rng.random()
            omega = rng.choice([1.0, 1.5, 1.9, 0.376])
            tol = 10 ** rng.uniform(-9, -2)
            K = rng.choice([1, 1, 2, 5])
            maxit = rng.choice([3000, 200, 37])
            if op < 0.2:
                k = rng.randint(0, 40)
                g.iterate(omega, k); oracle.iterate(ref, omega, k); log.append(("it", omega, k))
            elif op < 0.4:
                k = rng.randint(0, 40)
                g.jacobi(k); oracle.jacobi_iterate(ref, k); log.append(("jit", k))
            else:
                jac = op >= 0.7
                if jac:
                    r, rr = g.jacobi_solve(tol, maxit, K), oracle.jacobi_solve(ref, tol, maxit, K)
                else:
                    r, rr = g.solve(omega, tol, maxit, K), oracle.solve(ref, omega, tol, maxit, K)
                log.append(("jsolve" if jac else "solve", omega, tol, maxit, K, r.iters, rr.iters))
                if (r.converged, r.iters, r.max_change) != (rr.converged, rr.iters, rr.max_change):
                    bad += 1
                    print("MISMATCH", rows, cols, kernel, T, dtype, log, r, rr, flush=True)
                    break
        out = g.download()
    if not np.array_equal(out, ref.astype(np.float64)):
        bad += 1
        print("GRID MISMATCH", rows, cols, kernel, T, dtype, log, flush=True)
    n += 1
print(f"fuzz-mixed: {n} cases, {bad} bad, {time.time() - t0:.0f} s")
