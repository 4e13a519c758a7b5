"""Randomised differential test of the round-2 paths against the oracle
(development aid): single-slab and virtual (pushing) handles, f64 and f32,
SOR and Jacobi calls interleaved, iterate / solve / reset, all kernels and
depths (the skew-2 schedule, the persistent K6 launch, the deferred stop test
on slabs, exact re-runs).  Grids, iteration counts and reported maxima are
compared bitwise.  usage: python tools/fuzz_r2.py SECONDS SEED"""
import random
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402

budget = float(sys.argv[1])
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = random.Random(seed)
t0 = time.time()
n = bad = 0
KERNELS = [("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4), ("natural", 1)]
while time.time() - t0 < budget:
    nslabs = rng.choice([1, 1, 2, 3, 4])
    rows = rng.randint(max(1, 8 * nslabs), 360)
    cols = rng.randint(1, 640)
    kernel, T = rng.choice(KERNELS)
    if nslabs > 1 and rows // nslabs < 2 * T:
        kernel, T = "fused", 1
    dtype = rng.choice(["f64", "f64", "f32"])
    init = SI.random_edges(rows, cols, seed=rng.randint(0, 10 ** 6))
    ref = oracle.to_storage(init, dtype)
    log = []
    ok = True
    g = P.Grid.create(init, dtype=dtype) if nslabs == 1 else P.Grid.create_virtual(init, nslabs, dtype=dtype)
    try:
        g.set_kernel(kernel, T)
        for _ in range(rng.randint(1, 6)):
            op = rng.random()
            omega = rng.choice([1.0, 1.5, 1.9, 1.97, 0.376])
            jac = kernel != "natural" and rng.random() < 0.25
            if op < 0.3:
                k = rng.randint(0, 45)
                if jac:
                    g.jacobi(k)
                    oracle.jacobi_iterate(ref, k)
                else:
                    g.iterate(omega, k)
                    oracle.iterate(ref, omega, k)
                log.append(("jac" if jac else "it", omega, k))
            elif op < 0.4:
                g.reset(init)
                ref = oracle.to_storage(init, dtype)
                log.append(("reset",))
            else:
                tol = 10 ** rng.uniform(-9, -2)
                K = rng.choice([1, 1, 1, 2, 5])
                maxit = rng.choice([2500, 200, 37])
                if jac:
                    r = g.jacobi_solve(tol, maxit, K)
                    rr = oracle.jacobi_solve(ref, tol, maxit, K)
                else:
                    r = g.solve(omega, tol, maxit, K)
                    rr = oracle.solve(ref, omega, tol, maxit, K)
                log.append(("jsolve" if jac else "solve", omega, tol, maxit, K, r.iters, rr.iters))
                if (r.converged, r.iters, r.max_change) != (rr.status == 0, rr.iters, rr.max_change):
                    ok = False
                    print("MISMATCH", rows, cols, nslabs, dtype, kernel, T, log, r, rr, flush=True)
                    break
        if ok and not np.array_equal(g.download(), ref.astype(np.float64)):
            ok = False
            print("GRID MISMATCH", rows, cols, nslabs, dtype, kernel, T, log, flush=True)
    finally:
        g.close()
    bad += 0 if ok else 1
    n += 1
print(f"fuzz_r2 seed {seed}: {n} cases, {bad} bad, {time.time() - t0:.0f} s", flush=True)
