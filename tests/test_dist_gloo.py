"""Multi-rank host logic of the row-slab decomposition on CPU.

Two (and three) gloo ranks emulate the dist path's schedule with the oracle as
the per-slab compute: the partition is the library's `sor_partition_rows`
(host logic, no GPU), halo depth and exchange cadence are the library's
(1 row per half-sweep for K1; 2T rows per T-iteration pass for K3/K4), parity
follows the global row (row_off), and the max-change is joined with an
allreduce-MAX over ranks.  The gathered grid and the joined max must equal the
single-process oracle bitwise.  `-m "not gpu"`.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import sor_inputs as SI


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(u, lo, hi, g0, h, rank, world):
    """Send my first/last h owned rows to the neighbours' halos (library order)."""
    reqs = []
    top = torch.from_numpy(np.ascontiguousarray(u[lo - g0:lo - g0 + h]))
    bot = torch.from_numpy(np.ascontiguousarray(u[hi - g0 - h:hi - g0]))
    rtop = torch.empty_like(top)
    rbot = torch.empty_like(bot)
    if rank > 0:
        reqs.append(dist.isend(top, rank - 1))
        reqs.append(dist.irecv(rtop, rank - 1))
    if rank + 1 < world:
        reqs.append(dist.isend(bot, rank + 1))
        reqs.append(dist.irecv(rbot, rank + 1))
    for r in reqs:
        r.wait()
    if rank > 0:
        u[lo - g0 - h:lo - g0] = rtop.numpy()
    if rank + 1 < world:
        u[hi - g0:hi - g0 + h] = rbot.numpy()


def _worker(rank, world, port, mode, T, iters, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_1401_0763_b200 as P
    rows, cols = 61, 47
    init = SI.random_field(rows, cols, seed=17)
    lo, hi = P.partition_rows(rows, world, rank)
    h = 1 if mode == "k1" else 2 * T
    g0 = max(0, lo - h)                       # global row of local row 0
    g1 = min(rows + 2, hi + h)
    u = init[g0:g1].copy()
    omega = 1.83
    last_max = 0.0
    if mode == "k1":
        for k in range(iters):
            for c in (0, 1):
                old = u.copy()
                oracle.half_sweep(u, c, omega, row_off=g0)
                _exchange(u, lo, hi, g0, 1, rank, world)
                if k == iters - 1:
                    d = np.abs(u[lo - g0:hi - g0] - old[lo - g0:hi - g0]).max()
                    last_max = max(last_max, float(d))
    else:
        done = 0
        while done < iters:
            t = min(T, iters - done)
            old = u.copy()
            oracle.iterate(u, omega, t, row_off=g0)      # halo rows act as a fixed ring
            if done + t == iters:
                # the joined max-change is that of the LAST iteration: recompute it
                # from X_{k-1} on the owned rows (the ring rows stay correct for t-1)
                v = old.copy()
                if t > 1:
                    oracle.iterate(v, omega, t - 1, row_off=g0)
                last_max = float(np.abs(u[lo - g0:hi - g0] - v[lo - g0:hi - g0]).max())
            _exchange(u, lo, hi, g0, 2 * T, rank, world)
            done += t
    m = torch.tensor([last_max], dtype=torch.float64)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    # gather owned rows to rank 0 (ring rows come with the first/last slab)
    a = 0 if rank == 0 else lo
    b = rows + 2 if rank == world - 1 else hi
    part = torch.from_numpy(np.ascontiguousarray(u[a - g0:b - g0]))
    parts = [None] * world if rank == 0 else None
    dist.gather_object(part.numpy(), parts, dst=0)
    if rank == 0:
        out_q.put((np.concatenate(parts, axis=0), float(m.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,T,world", [("k1", 1, 2), ("wave", 1, 2), ("wave", 2, 2), ("wave", 3, 3),
                                          ("wave", 4, 2)])
def test_slab_schedule_matches_serial(orc, mode, T, world):
    import oracle
    iters = 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, T, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    grid, m = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = SI.random_field(61, 47, seed=17)
    rep = oracle.iterate(ref, 1.83, iters, measure_last=True)
    assert np.array_equal(grid, ref)
    assert m == rep.max_change
