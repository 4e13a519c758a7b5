"""Randomised differential test of K7 (SOR_KERNEL_RESIDENT) and the one-pass
3-D kernel against the oracle (development aid): random grid shapes (2-D up to
1100 x 1200, i.e. from one CTA to ~148 blocks; 3-D up to 40 x 60 x 200), random
depths, omegas, iterate / solve / reset sequences and kernel switches on one
handle; grids, iteration counts and reported maxima compared bitwise.
usage: python tools/fuzz_k7.py SECONDS SEED"""
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
while time.time() - t0 < budget:
    dtype = rng.choice(["f64", "f64", "f32"])
    if rng.random() < 0.75:
        rows = rng.choice([rng.randint(1, 100), rng.randint(50, 400), rng.randint(300, 1100)])
        cols = rng.choice([rng.randint(1, 126), rng.randint(100, 700), rng.randint(600, 1200)])
        init = SI.random_edges(rows, cols, seed=rng.randint(0, 10 ** 6))
        ref = oracle.to_storage(init, dtype)
        log = []
        with P.Grid.create(init, dtype=dtype) as g:
            for _ in range(rng.randint(1, 5)):
                T = rng.randint(1, 4)
                kern = rng.choice(["resident", "resident", "resident", "temporal"])
                g.set_kernel(kern, T)
                op = rng.random()
                omega = rng.choice([1.0, 1.5, 1.9, 1.97, 0.376])
                if op < 0.5:
                    k = rng.randint(0, 30)
                    want = rng.random() < 0.5
                    d = g.iterate(omega, k, want_delta=want)
                    rep = oracle.iterate(ref, omega, k, measure_last=want)
                    log.append(("it", kern, T, omega, k))
                    if want and k and d != rep.max_change:
                        bad += 1
                        print("MISMATCH delta", rows, cols, dtype, log, flush=True)
                elif op < 0.6:
                    g.reset(init)
                    ref = oracle.to_storage(init, dtype)
                    log.append(("reset",))
                elif rows * cols <= 200000:
                    tol = 10 ** rng.uniform(-8, -2)
                    K = rng.choice([1, 1, 3])
                    maxit = rng.choice([400, 50, 9])
                    r = g.solve(omega, tol, maxit, K)
                    rr = oracle.solve(ref, omega, tol, maxit, K)
                    log.append(("solve", kern, T, omega, tol, K, maxit))
                    if (r.converged, r.iters, r.max_change) != (rr.converged, rr.iters, rr.max_change):
                        bad += 1
                        print("MISMATCH solve", rows, cols, dtype, log, flush=True)
            if not np.array_equal(g.download(), ref.astype(np.float64)):
                bad += 1
                print("MISMATCH grid", rows, cols, dtype, log, flush=True)
    else:
        nz, ny, nx = rng.randint(1, 40), rng.randint(1, 60), rng.randint(1, 200)
        init = SI.random_field3d(nz, ny, nx, seed=rng.randint(0, 10 ** 6), lo=-10.0, hi=100.0)
        if rng.random() < 0.3:
            init = init * 1e-306
        ref = init.copy() if dtype == "f64" else init.astype(np.float32)
        log = []
        with P.Grid3D(init, dtype=dtype) as g:
            g.set_kernel(rng.choice(["fused", "fused", "natural"]))
            for _ in range(rng.randint(1, 3)):
                omega = rng.choice([1.0, 1.5, 1.8])
                if rng.random() < 0.6:
                    k = rng.randint(0, 20)
                    g.iterate(omega, k)
                    oracle.sor3d_iterate(ref, omega, k)
                    log.append(("it", omega, k))
                else:
                    tol, K, maxit = 10 ** rng.uniform(-8, -2), rng.choice([1, 2]), rng.choice([200, 30])
                    r = g.solve(omega, tol, maxit, K)
                    rr = oracle.sor3d_solve(ref, omega, tol, maxit, K)
                    log.append(("solve", omega, tol, K, maxit))
                    if (r.converged, r.iters, r.max_change) != (rr.converged, rr.iters, rr.max_change):
                        bad += 1
                        print("MISMATCH 3d solve", nz, ny, nx, dtype, log, flush=True)
            if not np.array_equal(g.download(), ref.astype(np.float64)):
                bad += 1
                print("MISMATCH 3d grid", nz, ny, nx, dtype, log, flush=True)
    n += 1
print(f"fuzz_k7 seed {seed}: {n} sequences, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
