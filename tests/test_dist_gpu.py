"""Multi-slab paths on the GPU, bitwise against the oracle.

* Virtual slabs (one process): the device-initiated halo push and its
  flags (HaloLink), the deferred stop test on slabs, Jacobi on slabs,
  changes of T between passes (strip layouts of producer and consumer
  differ), and the copy-exchange fallback (SOR_VIRTUAL_COPY=1).
* Dist over CUDA IPC, 2-4 processes sharing the one GPU of the test box:
  the real rendezvous, IPC mappings, rank-0 scatter (init=None elsewhere),
  peer pushes into another process's memory, the cross-rank max join, the
  gather (download / download_rows) and reset.  Ranks that share a GPU run
  in lockstep (a host barrier between passes), because kernels of different
  processes on one device must never wait on each other.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import sor_inputs as SI

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gpu(sor):
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    torch.cuda.set_device(0)
    return sor


def _ref(orc, init, dtype, fn):
    u = orc.to_storage(init, dtype)
    r = fn(u)
    return u.astype(np.float64), r


@pytest.mark.parametrize("nslabs", [2, 3, 5])
@pytest.mark.parametrize("T", [1, 2, 3, 4])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_virtual_jacobi(gpu, orc, nslabs, T, dtype):
    init = SI.random_field(157, 290, seed=nslabs * 10 + T, lo=-20.0, hi=80.0)
    ref, rep = _ref(orc, init, dtype, lambda u: orc.jacobi_iterate(u, 13, measure_last=True))
    with gpu.Grid.create_virtual(init, nslabs, dtype=dtype) as g:
        g.set_kernel("temporal" if T > 1 else "fused", T)
        d = g.jacobi(13, want_delta=True)
        out = g.download()
    assert np.array_equal(out, ref) and d == rep.max_change
    ref2, rep2 = _ref(orc, init, dtype, lambda u: orc.jacobi_solve(u, 1e-3, 3000, 1))
    with gpu.Grid.create_virtual(init, nslabs, dtype=dtype) as g:
        g.set_kernel("temporal" if T > 1 else "fused", T)
        r = g.jacobi_solve(1e-3, 3000, 1)
        out = g.download()
    assert (r.converged, r.iters, r.max_change) == (rep2.status == 0, rep2.iters, rep2.max_change)
    assert np.array_equal(out, ref2)


@pytest.mark.parametrize("nslabs", [2, 4])
@pytest.mark.parametrize("T", [1, 2, 3, 4])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_virtual_deferred_solve(gpu, orc, nslabs, T, dtype):
    """Slabs with the deferred stop test (third plane, decision block in the
    first slab's launch), exact re-runs, then continuation on the handle."""
    init = SI.random_edges(180, 300, seed=60 + T)
    ref, rr = _ref(orc, init, dtype, lambda u: orc.solve(u, 1.93, 1e-6, 20000, 1))
    with gpu.Grid.create_virtual(init, nslabs, dtype=dtype) as g:
        g.set_kernel("temporal" if T > 1 else "fused", T)
        r = g.solve(1.93, 1e-6, 20000, 1)
        assert (r.converged, r.iters, r.max_change) == (rr.status == 0, rr.iters, rr.max_change)
        assert np.array_equal(g.download(), ref)
        g.iterate(1.93, 5)
        r2 = g.solve(1.93, 1e-8, 20000, 3)
        out = g.download()
    u = orc.to_storage(ref, dtype)
    orc.iterate(u, 1.93, 5)
    rr2 = orc.solve(u, 1.93, 1e-8, 20000, 3)
    assert (r2.converged, r2.iters, r2.max_change) == (rr2.status == 0, rr2.iters, rr2.max_change)
    assert np.array_equal(out, u.astype(np.float64))


def test_virtual_depth_changes_between_calls(gpu, orc):
    """Consecutive passes of different depth (remainders, set_kernel) and
    method: the consumer's strip layout differs from the producer's."""
    init = SI.random_field(200, 410, seed=3, lo=-10.0, hi=10.0)
    u = init.copy()
    with gpu.Grid.create_virtual(init, 4) as g:
        for T, n, jac in ((4, 9, False), (1, 3, False), (3, 7, True), (2, 5, False), (4, 6, True), (3, 10, False)):
            g.set_kernel("temporal" if T > 1 else "fused", T)
            if jac:
                g.jacobi(n)
                orc.jacobi_iterate(u, n)
            else:
                g.iterate(1.77, n)
                orc.iterate(u, 1.77, n)
            assert np.array_equal(g.download(), u), (T, n, jac)


_COPY = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import oracle, sor_inputs as SI, paper_1401_0763_b200 as P
init = SI.random_field(203, 150, seed=5, lo=-5.0, hi=5.0)
for T in (1, 2, 4):
    ref = init.copy(); rr = oracle.solve(ref, 1.9, 1e-6, 5000, 1)
    with P.Grid.create_virtual(init, 3) as g:
        g.set_kernel("temporal" if T > 1 else "fused", T)
        r = g.solve(1.9, 1e-6, 5000, 1)
        assert (r.iters, r.max_change) == (rr.iters, rr.max_change), (T, r, rr.iters)
        assert np.array_equal(g.download(), ref), T
        assert g.stats["halo_exchanges"] > 0
print("ok")
"""


def test_virtual_copy_exchange_fallback(gpu):
    r = subprocess.run([sys.executable, "-c", _COPY % ROOT], env=dict(os.environ, SOR_VIRTUAL_COPY="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-3000:]


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_dist_ipc_processes(gpu, nranks):
    """nranks processes, one dist-IPC handle (rank 0 holds the init), every
    collective call of the ABI, bitwise against the oracle (rank 0)."""
    uid = gpu.ipc_unique_id().rstrip(b"\0")
    worker = os.path.join(ROOT, "tests", "dist_ipc_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(nranks), str(r), uid.ljust(128, b"\0").hex(), "0"],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(nranks)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=900))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    log = outs[0][0]
    assert "DONE fails=0" in log, log + "\n" + "\n".join(o[1][-2000:] for o in outs)
    assert all(p.returncode == 0 for p in procs), [o[1][-2000:] for o in outs]
    assert log.count("ok  ") >= 25


@pytest.mark.parametrize("nranks,seed", [(2, 41), (3, 42)])
def test_dist_ipc_random_sequences(gpu, nranks, seed):
    """Random collective call sequences on dist-IPC handles (shapes, dtypes,
    depths, SOR/Jacobi, iterate/solve/reset/download_rows), every rank a
    process on the one GPU, rank 0 bitwise against the oracle
    (tools/fuzz_dist_ipc.py)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_dist_ipc.py"), "launch", str(nranks), "12",
                        str(seed)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "0 bad" in r.stdout, r.stdout[-3000:]
