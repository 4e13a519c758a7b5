"""Randomised differential test of the NEXT-4 variants (multi-colour and block
red-black SOR) and the deep temporal depths (T = 5, 6) against the oracle
(development aid): random shapes from one cell to several tiles, random
colourings (ca, cb, nc) and block sizes, variant iterate / solve calls
interleaved with red-black SOR calls at every kernel and depth, Jacobi calls and
resets on one handle (the variants share the handle's planes and the deferred
solve's third plane).  Grids, iteration counts and reported maxima are compared
bitwise.  usage: python tools/fuzz_next4.py SECONDS SEED"""
import math
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
KERNELS = [("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4), ("temporal", 5), ("temporal", 6),
           ("natural", 1)]


def draw_variant():
    if rng.random() < 0.5:
        nc = rng.randint(2, 8)
        while True:
            ca, cb = rng.randint(-7, 9), rng.randint(-7, 9)
            if ca % nc and cb % nc:
                return ("mc", ca, cb, nc)
    return ("bp", rng.choice([1, 2, 3, 4, 5, 7, 8, 11, 16, 23, 32]))


while time.time() - t0 < budget:
    rows = rng.choice([rng.randint(1, 40), rng.randint(1, 420)])
    cols = rng.choice([rng.randint(1, 40), rng.randint(1, 700)])
    kernel, T = rng.choice(KERNELS)
    dtype = rng.choice(["f64", "f64", "f32"])
    fld = rng.random() < 0.5
    s0 = rng.randint(0, 10 ** 6)
    init = SI.random_field(rows, cols, seed=s0, lo=-50.0, hi=100.0) if fld else SI.random_edges(rows, cols, seed=s0)
    ref = oracle.to_storage(init, dtype)
    log = []
    ok = True
    g = P.Grid.create(init, dtype=dtype)
    try:
        g.set_kernel(kernel, T)
        for _ in range(rng.randint(1, 6)):
            op = rng.random()
            omega = rng.choice([1.0, 1.5, 1.9, 1.97, 0.376])
            which = rng.random()
            v = draw_variant() if which < 0.6 else None
            jac = v is None and kernel != "natural" and T <= 4 and which < 0.7
            if v is not None:
                pv = P.Variant.multicolor(*v[1:]) if v[0] == "mc" else P.Variant.blocks(v[1])
            if op < 0.4:
                k = rng.randint(0, 25)
                if v is not None:
                    d = g.variant_iterate(pv, omega, k, want_delta=True)
                    rr = (oracle.multicolor_iterate(ref, omega, k, *v[1:], measure_last=True) if v[0] == "mc"
                          else oracle.block_iterate(ref, omega, k, v[1], measure_last=True))
                    if k > 0 and d != rr.max_change:
                        ok = False
                        print("DELTA MISMATCH", rows, cols, dtype, kernel, T, v, log, d, rr.max_change, flush=True)
                        break
                elif jac:
                    g.jacobi(k)
                    oracle.jacobi_iterate(ref, k)
                else:
                    g.iterate(omega, k)
                    oracle.iterate(ref, omega, k)
                log.append((v or ("jac" if jac else "it"), omega, k))
            elif op < 0.5:
                g.reset(init)
                ref = oracle.to_storage(init, dtype)
                log.append(("reset",))
            else:
                tol = 10 ** rng.uniform(-9, -1)
                K = rng.choice([1, 1, 1, 2, 5])
                maxit = rng.choice([1500, 200, 37])
                if v is not None:
                    r = g.variant_solve(pv, omega, tol, maxit, K)
                    rr = (oracle.multicolor_solve(ref, omega, tol, maxit, K, *v[1:]) if v[0] == "mc"
                          else oracle.block_solve(ref, omega, tol, maxit, v[1], K))
                elif jac:
                    r = g.jacobi_solve(tol, maxit, K)
                    rr = oracle.jacobi_solve(ref, tol, maxit, K)
                else:
                    r = g.solve(omega, tol, maxit, K)
                    rr = oracle.solve(ref, omega, tol, maxit, K)
                log.append((v or ("jsolve" if jac else "solve"), omega, tol, maxit, K, r.iters, rr.iters))
                same = (r.converged, r.iters) == (rr.status == 0, rr.iters) and (
                    r.max_change == rr.max_change or (math.isnan(r.max_change) and math.isnan(rr.max_change)))
                if not same:
                    ok = False
                    print("MISMATCH", rows, cols, dtype, kernel, T, log, r, rr, flush=True)
                    break
            if rng.random() < 0.3 and not np.array_equal(g.download(), ref.astype(np.float64)):
                ok = False
                print("GRID MISMATCH (mid)", rows, cols, dtype, kernel, T, log, flush=True)
                break
        if ok and not np.array_equal(g.download(), ref.astype(np.float64)):
            ok = False
            print("GRID MISMATCH", rows, cols, dtype, kernel, T, log, flush=True)
    finally:
        g.close()
    bad += 0 if ok else 1
    n += 1
print(f"fuzz_next4 seed {seed}: {n} cases, {bad} bad, {time.time() - t0:.0f} s", flush=True)
