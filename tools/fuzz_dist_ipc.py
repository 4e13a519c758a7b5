"""Randomised differential test of dist-IPC handles (one process per rank; all
ranks on one GPU run in lockstep).  Every rank draws the same
random call sequence (shapes, dtypes, kernels, depths, SOR/Jacobi, iterate /
solve / reset / download / download_rows); rank 0 holds the init and compares
every result with the CPU oracle, bitwise.

usage: python tools/fuzz_dist_ipc.py launch NRANKS NCASES SEED   (spawns the ranks)
       python tools/fuzz_dist_ipc.py rank NRANKS RANK NCASES SEED IDHEX
"""
import os
import random
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402


def rank_main(nranks, rank, seconds, seed, uid):
    orc = None
    if rank == 0:
        import oracle as orc
    rng = random.Random(seed)
    t0 = time.time()
    n = bad = 0
    # every rank runs the same number of cases (a time budget could end the
    # ranks at different cases, and their collective calls would not match)
    ncases = max(1, int(seconds))
    for case in range(ncases):
        rows = rng.randint(8 * nranks, 220)
        cols = rng.randint(1, 400)
        dtype = rng.choice(["f64", "f64", "f32"])
        kernel, T = rng.choice([("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4)])
        if rows // nranks < 2 * T:
            kernel, T = "fused", 1
        init = SI.random_edges(rows, cols, seed=rng.randint(0, 10 ** 6))
        g = P.Grid.create_dist_ipc(init if rank == 0 else None, rank, nranks, 0, uid, dtype=dtype, rows=rows,
                                   cols=cols)
        g.set_kernel(kernel, T)
        ref = orc.to_storage(init, dtype) if rank == 0 else None
        log = []
        ok = True
        for _ in range(rng.randint(1, 5)):
            op = rng.random()
            omega = rng.choice([1.0, 1.5, 1.9, 1.97, 0.376])
            jac = rng.random() < 0.2
            if op < 0.3:
                k = rng.randint(0, 30)
                if jac:
                    g.jacobi(k)
                    if rank == 0:
                        orc.jacobi_iterate(ref, k)
                else:
                    g.iterate(omega, k)
                    if rank == 0:
                        orc.iterate(ref, omega, k)
                log.append(("jac" if jac else "it", omega, k))
            elif op < 0.4:
                g.reset(init if rank == 0 else None)
                if rank == 0:
                    ref = orc.to_storage(init, dtype)
                log.append(("reset",))
            elif op < 0.5:
                a = rng.randint(0, rows + 1)
                b = rng.randint(a + 1, rows + 2)
                out = g.download_rows(a, b)
                if rank == 0 and not np.array_equal(out, ref.astype(np.float64)[a:b]):
                    ok = False
                    print("ROWS MISMATCH", case, rows, cols, dtype, kernel, T, log, (a, b), flush=True)
                log.append(("rows", a, b))
            else:
                tol = 10 ** rng.uniform(-8, -2)
                K = rng.choice([1, 1, 2, 5])
                maxit = rng.choice([600, 120, 37])
                if jac:
                    r = g.jacobi_solve(tol, maxit, K)
                    rr = orc.jacobi_solve(ref, tol, maxit, K) if rank == 0 else None
                else:
                    r = g.solve(omega, tol, maxit, K)
                    rr = orc.solve(ref, omega, tol, maxit, K) if rank == 0 else None
                log.append(("jsolve" if jac else "solve", omega, tol, maxit, K, r.iters))
                if rank == 0 and (r.converged, r.iters, r.max_change) != (rr.status == 0, rr.iters, rr.max_change):
                    ok = False
                    print("SOLVE MISMATCH", case, rows, cols, dtype, kernel, T, log, r, rr.iters, flush=True)
        out = g.download()
        if rank == 0 and not np.array_equal(out, ref.astype(np.float64)):
            ok = False
            print("GRID MISMATCH", case, rows, cols, dtype, kernel, T, log, flush=True)
        g.close()
        n += 1
        bad += 0 if ok else 1
    if rank == 0:
        print(f"fuzz_dist_ipc nranks {nranks} seed {seed}: {n} cases, {bad} bad, {time.time() - t0:.0f} s",
              flush=True)
    return bad


def launch(nranks, seconds, seed):
    uid = P.ipc_unique_id().rstrip(b"\0").ljust(128, b"\0").hex()
    me = os.path.abspath(__file__)
    procs = [subprocess.Popen([sys.executable, me, "rank", str(nranks), str(r), str(seconds), str(seed), uid])
             for r in range(nranks)]
    rc = [p.wait() for p in procs]
    return max(rc)


if __name__ == "__main__":
    if sys.argv[1] == "launch":
        sys.exit(launch(int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])))
    nr, rk, sec, sd, idhex = int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
    sys.exit(1 if rank_main(nr, rk, sec, sd, bytes.fromhex(idhex)) else 0)
