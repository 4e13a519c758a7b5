"""One rank of a dist-IPC handle (run as a process by tests/test_dist_gpu.py).

Usage: python dist_ipc_worker.py NRANKS RANK IPC_ID_HEX DEVICE
Every rank runs the same sequence of collective calls; rank 0 holds the
init, compares every download with the CPU oracle (test infrastructure,
allowed here) and prints one line per checked case.  Exit code 0 iff every
comparison was bitwise equal.  All ranks share one GPU in the test, so the
library runs them in lockstep.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402


def main():
    nranks, rank, uid_hex, device = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
    uid = bytes.fromhex(uid_hex)
    orc = None
    if rank == 0:
        import oracle as orc
    fails = []

    def check(name, got, ref, d=None, dref=None):
        if rank != 0:
            return
        ok = np.array_equal(got, ref) and (d is None or d == dref)
        print(f"{'ok  ' if ok else 'FAIL'} {name}", flush=True)
        if not ok:
            fails.append(name)

    def mk(init, rows, cols, dtype):
        return P.Grid.create_dist_ipc(init if rank == 0 else None, rank, nranks, device, uid,
                                      dtype=dtype, rows=rows, cols=cols)

    # uneven slabs (203 = 3*67+2, odd first rows), several strips (150 columns)
    rows, cols = 203, 150
    for dtype in ("f64", "f32"):
        init = SI.random_field(rows, cols, seed=7, lo=-50.0, hi=100.0)
        g = mk(init, rows, cols, dtype)
        for T in (1, 2, 3, 4):
            g.set_kernel("temporal" if T > 1 else "fused", T)
            g.reset(init if rank == 0 else None)
            d = g.iterate(1.9, 11, want_delta=True)
            out = g.download()
            ref = dref = None
            if rank == 0:
                ref = orc.to_storage(init, dtype)
                dref = orc.iterate(ref, 1.9, 11, measure_last=True).max_change
                ref = ref.astype(np.float64)
            check(f"iterate {dtype} T={T}", out, ref, d, dref)
            # continuation with a solve (K=1: every iteration checked, deferred
            # decisions off in lockstep, exact re-runs of T-deep passes)
            r = g.solve(1.9, 1e-6, 4000, 1)
            out = g.download()
            rows_out = g.download_rows(50, 120)
            if rank == 0:
                u = orc.to_storage(init, dtype)
                orc.iterate(u, 1.9, 11)
                rr = orc.solve(u, 1.9, 1e-6, 4000, 1)
                u = u.astype(np.float64)
                check(f"solve K=1 {dtype} T={T} ({r.iters} vs {rr.iters})", out, u,
                      (r.converged, r.iters, r.max_change), (rr.converged, rr.iters, rr.max_change))
                check(f"download_rows {dtype} T={T}", rows_out, u[50:120])
        # K > 1 cadence and maxit exhaustion
        g.set_kernel("temporal", 3)
        g.reset(init if rank == 0 else None)
        r = g.solve(1.7, 1e-300, 40, 7)
        out = g.download()
        if rank == 0:
            u = orc.to_storage(init, dtype)
            rr = orc.solve(u, 1.7, 1e-300, 40, 7)
            check(f"solve K=7 maxit {dtype}", out, u.astype(np.float64),
                  (r.converged, r.iters, r.max_change), (rr.converged, rr.iters, rr.max_change))
        # Jacobi on the same slabs
        g.set_kernel("temporal", 2)
        g.reset(init if rank == 0 else None)
        d = g.jacobi(9, want_delta=True)
        out = g.download()
        if rank == 0:
            u = orc.to_storage(init, dtype)
            rj = orc.jacobi_iterate(u, 9, measure_last=True)
            check(f"jacobi {dtype} T=2", out, u.astype(np.float64), d, rj.max_change)
        st = g.stats
        if rank == 0:
            print(f"stats rank0 {st['row_lo']}..{st['row_hi']} nranks {st['nranks']}", flush=True)
        g.close()
    # C1 solve on the slabs (the BJ configs[0] problem)
    cfg = SI.config("C1")
    g = mk(cfg.init(), 64, 64, "f64")
    g.set_kernel("temporal", 2)
    r = g.solve(cfg.omega, cfg.tol, cfg.maxit, 1)
    out = g.download()
    if rank == 0:
        u = cfg.init()
        rr = orc.solve(u, cfg.omega, cfg.tol, cfg.maxit, 1)
        check(f"C1 solve ({r.iters})", out, u, (r.iters, r.max_change), (rr.iters, rr.max_change))
    g.close()
    if rank == 0:
        print("DONE fails=%d" % len(fails), flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
