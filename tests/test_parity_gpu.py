"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element, on the same seeded inputs (`-m gpu`, needs a B200).

The bar (BASELINE.json north_star): with the canonical
operation order and no contraction on both sides every variant is expected
BITWISE equal to the oracle; the tests assert bitwise equality, which implies
the stated tolerances (fp64 <= 1e-12*max|bnd|, fp32 <= 1e-5 rel, iterations
+-1).  Sizes span several warp strips (124..112 columns) and bands, with
ragged tails, odd/even dimensions and degenerate 1-wide grids.
"""
import os

import numpy as np
import pytest

import sor_inputs as SI

pytestmark = pytest.mark.gpu

KERNELS = [("natural", 1), ("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4),
           ("resident", 1), ("resident", 2), ("resident", 3), ("resident", 4)]
SIZES = [(1, 1), (1, 9), (7, 1), (2, 2), (3, 5), (8, 8), (31, 33), (64, 64), (65, 127),
         (130, 257), (257, 130), (300, 517)]


@pytest.fixture(scope="module")
def gpu(sor):
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    torch.cuda.set_device(0)
    return sor


def _field(rows, cols, seed, dtype):
    u = SI.random_field(rows, cols, seed=seed, lo=-50.0, hi=100.0)
    return u


def _oracle_iterate(orc, init, dtype, omega, iters, measure_last=False):
    u = orc.to_storage(init, dtype)
    rep = orc.iterate(u, omega, iters, measure_last=measure_last)
    return u.astype(np.float64), rep


@pytest.mark.parametrize("kernel,T", KERNELS)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("rows,cols", SIZES)
def test_iterate_bitwise(gpu, orc, kernel, T, dtype, rows, cols):
    init = _field(rows, cols, seed=rows * 1000 + cols, dtype=dtype)
    iters = 7                                   # not a multiple of T: remainder passes
    ref, rep = _oracle_iterate(orc, init, dtype, 1.7, iters, measure_last=True)
    with gpu.Grid.create(init, dtype=dtype) as g:
        g.set_kernel(kernel, T)
        d = g.iterate(1.7, iters, want_delta=True)
        out = g.download()
    assert np.array_equal(out, ref), np.abs(out - ref).max()
    assert d == rep.max_change


@pytest.mark.parametrize("kernel,T", KERNELS)
def test_iterate_many_omegas_and_continuation(gpu, orc, kernel, T):
    init = _field(97, 250, seed=5, dtype="f64")
    ref = init.copy()
    with gpu.Grid.create(init) as g:
        g.set_kernel(kernel, T)
        for omega, n in ((0.376, 3), (1.0, 5), (1.5, 4), (1.99, 9), (1.2, 0), (1.93, 1)):
            orc.iterate(ref, omega, n)
            g.iterate(omega, n)
        out = g.download()
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("kernel,T", KERNELS + [("small", 1)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c1_solve_exact(gpu, orc, kernel, T, dtype):
    """BJ configs[0]: iterations-to-tolerance and final grid equal to the oracle."""
    cfg = SI.config("C1")
    ref = orc.to_storage(cfg.init(), dtype)
    rr = orc.solve(ref, cfg.omega, cfg.tol, cfg.maxit, 1)
    with gpu.Grid.create(cfg.init(), dtype=dtype) as g:
        g.set_kernel(kernel, T)
        r = g.solve(cfg.omega, cfg.tol, cfg.maxit, 1)
        out = g.download()
    assert r.converged == rr.converged and r.iters == rr.iters
    assert r.max_change == rr.max_change
    assert np.array_equal(out, ref.astype(np.float64))


@pytest.mark.parametrize("kernel,T", KERNELS)
@pytest.mark.parametrize("K", [1, 3, 8])
def test_solve_cadence_and_not_converged(gpu, orc, kernel, T, K):
    init = SI.random_edges(50, 77, seed=K)
    ref = init.copy()
    rr = orc.solve(ref, 1.8, 1e-3, 173, check_every=K)
    with gpu.Grid.create(init) as g:
        g.set_kernel(kernel, T)
        r = g.solve(1.8, 1e-3, 173, check_every=K)
        out = g.download()
        st = g.stats
    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
    assert np.array_equal(out, ref)
    assert st["half_sweeps"] == 2 * rr.iters
    # maxit reached
    ref2 = init.copy()
    rr2 = orc.solve(ref2, 1.8, 1e-30, 20, check_every=K)
    with gpu.Grid.create(init) as g:
        g.set_kernel(kernel, T)
        r2 = g.solve(1.8, 1e-30, 20, check_every=K)
        out2 = g.download()
    assert not r2.converged and r2.iters == 20 and rr2.iters == 20
    assert r2.max_change == rr2.max_change
    assert np.array_equal(out2, ref2)


def test_solve_then_continue(gpu, orc):
    cfg = SI.config("C1")
    ref = cfg.init()
    orc.iterate(ref, cfg.omega, 100)
    rr = orc.solve(ref, cfg.omega, 1e-5, 10000, 1)
    with gpu.Grid.create(cfg.init()) as g:
        g.iterate(cfg.omega, 100)
        r = g.solve(cfg.omega, 1e-5, 10000, 1)
        out = g.download()
    assert r.iters == rr.iters and np.array_equal(out, ref)


@pytest.mark.parametrize("nslabs", [2, 3, 4, 8])
@pytest.mark.parametrize("kernel,T", KERNELS)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_virtual_slabs_bitwise(gpu, orc, nslabs, kernel, T, dtype):
    """Row-slab decomposition (same kernels, halos, partition as dist mode)."""
    init = _field(203, 150, seed=nslabs, dtype=dtype)
    ref, rep = _oracle_iterate(orc, init, dtype, 1.9, 11, measure_last=True)
    with gpu.Grid.create_virtual(init, nslabs, dtype=dtype) as g:
        g.set_kernel(kernel, T)
        d = g.iterate(1.9, 11, want_delta=True)
        out = g.download()
    assert np.array_equal(out, ref)
    assert d == rep.max_change


@pytest.mark.parametrize("nslabs", [2, 5])
def test_virtual_slabs_solve(gpu, orc, nslabs):
    init = SI.random_edges(120, 90, seed=11)
    ref = init.copy()
    rr = orc.solve(ref, 1.9, 1e-6, 5000, 1)
    with gpu.Grid.create_virtual(init, nslabs) as g:
        r = g.solve(1.9, 1e-6, 5000, 1)
        out = g.download()
    assert r.iters == rr.iters and r.max_change == rr.max_change
    assert np.array_equal(out, ref)


def test_device_pointers_and_reset(gpu, orc):
    import torch
    init = SI.random_edges(200, 333, seed=9)
    ref = init.copy()
    orc.iterate(ref, 1.6, 13)
    dinit = torch.from_numpy(init).cuda()
    dout = torch.empty_like(dinit)
    with gpu.Grid.create(dinit) as g:
        g.iterate(1.6, 5)
        g.reset(dinit)                     # back to X_0
        g.iterate(1.6, 13)
        g.download(dout)
        rows = g.download_rows(50, 61)
    assert np.array_equal(dout.cpu().numpy(), ref)
    assert np.array_equal(rows, ref[50:61])


def test_device_init_written_by_pending_gpu_work(gpu, orc):
    """A device-resident init is read after the caller's pending work on other
    streams (sor.h: create / reset order their reads after it): the tensor is
    filled by asynchronous GPU work queued behind ~10 ms of kernels, and create
    / reset are called at once."""
    import torch
    init = SI.random_edges(300, 517, seed=21)
    ref = init.copy()
    orc.iterate(ref, 1.7, 9)
    pinned = torch.from_numpy(init).pin_memory()
    ballast = torch.empty(1 << 27, dtype=torch.float32, device="cuda")
    for use_reset in (False, True):
        dinit = torch.zeros(init.shape, dtype=torch.float64, device="cuda")
        g0 = gpu.Grid.create(np.zeros_like(init)) if use_reset else None
        torch.cuda.synchronize()
        for _ in range(12):
            ballast.normal_()                       # keeps the current stream busy
        dinit.copy_(pinned, non_blocking=True)      # the fill, queued behind it
        g = g0 if use_reset else gpu.Grid.create(dinit)
        if use_reset:
            g.reset(dinit)
        with g:
            g.set_kernel("temporal", 3)
            g.iterate(1.7, 9)
            out = g.download()
        assert np.array_equal(out, ref), use_reset


def test_external_stream(gpu, orc):
    import torch
    init = SI.random_edges(64, 300, seed=2)
    ref = init.copy()
    orc.iterate(ref, 1.5, 6)
    s = torch.cuda.Stream()
    with gpu.Grid.create(init) as g:
        g.set_stream(s.cuda_stream)
        g.iterate(1.5, 6)
        g.set_stream(None)
        out = g.download()
    assert np.array_equal(out, ref)


def test_wrong_shaped_buffers_are_rejected_by_the_binding(gpu, orc):
    """reset / download / download_rows with a buffer of the wrong shape or
    dtype raise before the C call (which would read or write out of bounds);
    the handle stays usable and unchanged."""
    init = SI.random_edges(20, 33, seed=4)
    ref = init.copy()
    orc.iterate(ref, 1.5, 3)
    with gpu.Grid.create(init) as g:
        g.iterate(1.5, 3)
        for bad in (lambda: g.reset(np.zeros((22, 34))), lambda: g.reset(np.zeros((35, 22))),
                    lambda: g.download(np.zeros((22, 36))), lambda: g.download(np.zeros(22 * 35)),
                    lambda: g.download_rows(3, 9, np.zeros((5, 35))), lambda: g.download_rows(3, 9, np.zeros((6, 34)))):
            with pytest.raises(ValueError):
                bad()
        with pytest.raises(TypeError):
            g.download(np.zeros((22, 35), dtype=np.float32))
        assert np.array_equal(g.download(), ref)
    with gpu.Grid3D(SI.random_field3d(4, 5, 6, seed=1)) as g3:
        with pytest.raises(ValueError):
            g3.download(np.zeros((6, 7, 9)))
        with pytest.raises(TypeError):
            g3.download(np.zeros((6, 7, 8), dtype=np.float32))
        assert g3.download().shape == (6, 7, 8)


def test_invalid_calls_leave_handle_usable(gpu):
    init = SI.north_hot(10, 10, 1.0)
    with gpu.Grid.create(init) as g:
        for bad in (lambda: g.iterate(2.0, 1), lambda: g.iterate(0.0, 1), lambda: g.iterate(1.0, -1),
                    lambda: g.solve(1.5, 0.0, 10), lambda: g.solve(1.5, 1e-3, 10, 11),
                    lambda: g.set_kernel("temporal", 7), lambda: g.set_kernel(99)):
            with pytest.raises(gpu.SorError) as e:
                bad()
            assert e.value.code == gpu.SOR_E_INVAL
        g.iterate(1.5, 2)
    bad = init.copy()
    bad[3, 3] = np.inf
    with pytest.raises(gpu.SorError):
        gpu.Grid.create(bad)
    big = SI.north_hot(400, 400, 1.0)
    with gpu.Grid.create(big) as g:
        with pytest.raises(gpu.SorError) as e:
            g.set_kernel("small")
        assert e.value.code == gpu.SOR_E_UNSUPPORTED


def test_zero_iterations_and_stats(gpu):
    init = SI.north_hot(30, 30, 1.0)
    with gpu.Grid.create(init) as g:
        assert g.iterate(1.5, 0, want_delta=True) == 0.0
        assert np.array_equal(g.download(), init)
        g.set_kernel("temporal", 4)
        g.iterate(1.5, 10)
        st = g.stats
        assert st["half_sweeps"] == 20 and st["hbm_passes"] == 3   # 2 + 4 + 4
        # the remainder pass, then both full passes in one persistent (K6) launch
        assert st["kernel_launches"] == (3 if os.environ.get("SOR_NO_PERSIST") else 2)
        assert g.elapsed_ms > 0


@pytest.mark.parametrize("T", [2, 3, 4])
@pytest.mark.parametrize("nudge", ["converge_here", "tie_continue"])
def test_solve_high_word_tie_resolved_exactly(gpu, orc, T, nudge):
    """ck=3 passes decide '<' on the high 32 bits; a tie must be resolved exactly."""
    init = SI.random_edges(60, 75, seed=21)
    probe = init.copy()
    hist = [orc.iterate(probe, 1.9, 1, measure_last=True).max_change for _ in range(60)]
    k = 41                                     # an iteration inside a pass
    m = hist[k - 1]
    assert min(hist[:k - 1]) > m               # no earlier iteration is below m
    tol = float(np.nextafter(m, np.inf)) if nudge == "converge_here" else m
    ref = init.copy()
    rr = orc.solve(ref, 1.9, tol, 500, 1)
    if nudge == "converge_here":
        assert rr.converged and rr.iters == k
    with gpu.Grid.create(init) as g:
        g.set_kernel("temporal", T)
        r = g.solve(1.9, tol, 500, 1)
        out = g.download()
    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("kernel,T", [("fused", 1), ("temporal", 3), ("natural", 1)])
def test_dist_single_rank_nccl(gpu, orc, kernel, T):
    """sor_create_dist with nranks=1: NCCL communicator, allreduce-max + finalize path."""
    init = SI.random_edges(90, 130, seed=31)
    ref = init.copy()
    orc.iterate(ref, 1.7, 10)
    rr = orc.solve(ref, 1.7, 1e-4, 3000, 2)
    uid = gpu.nccl_unique_id()
    with gpu.Grid.create_dist(init, 0, 1, 0, uid) as g:
        g.set_kernel(kernel, T)
        g.iterate(1.7, 10)
        r = g.solve(1.7, 1e-4, 3000, 2)
        out = g.download()
        st = g.stats
    assert (st["rank"], st["nranks"]) == (0, 1)
    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("T", [1, 2, 3, 4])
def test_deferred_solve_repeated_on_one_handle(gpu, orc, T):
    """Deferred stop test: the stop flag changes while a launch runs; repeated
    solves (reset in between), iterate/solve alternation and a re-run after an
    inconclusive probe all keep the oracle's iteration count and grid."""
    init = SI.random_edges(300, 517, seed=40 + T)
    ref = init.copy()
    rr = orc.solve(ref, 1.95, 1e-7, 20000, 1)
    with gpu.Grid.create(init) as g:
        g.set_kernel("temporal" if T > 1 else "fused", T)
        for _ in range(3):
            g.reset(init)
            r = g.solve(1.95, 1e-7, 20000, 1)
            assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
            assert np.array_equal(g.download(), ref)
        # continuation: a few more iterations, then a tighter solve on the same handle
        ref2 = ref.copy()
        orc.iterate(ref2, 1.95, 7)
        rr2 = orc.solve(ref2, 1.95, 1e-9, 20000, 1)
        g.iterate(1.95, 7)
        r2 = g.solve(1.95, 1e-9, 20000, 1)
        assert (r2.converged, r2.iters, r2.max_change) == (rr2.converged, rr2.iters, rr2.max_change)
        assert np.array_equal(g.download(), ref2)


_SUBPROC = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import oracle, sor_inputs as SI, paper_1401_0763_b200 as P
cfg = SI.config("C1")
ref = cfg.init(); rr = oracle.solve(ref, cfg.omega, cfg.tol, cfg.maxit, 1)
for kernel, T in (("fused", 1), ("temporal", 2), ("temporal", 4)):
    with P.Grid.create(cfg.init()) as g:
        g.set_kernel(kernel, T)
        r = g.solve(cfg.omega, cfg.tol, cfg.maxit, 1)
        assert (r.iters, r.max_change) == (rr.iters, rr.max_change), (kernel, T, r, rr.iters)
        assert np.array_equal(g.download(), ref), (kernel, T)
init = SI.random_edges(97, 260, seed=5)
ref = init.copy(); oracle.iterate(ref, 1.8, 9)
with P.Grid.create(init) as g:
    g.set_kernel("temporal", 3); g.iterate(1.8, 9)
    assert np.array_equal(g.download(), ref)
print("ok")
"""


@pytest.mark.parametrize("env", ["SOR_NO_DEFER", "SOR_NO_PDL", "SOR_NO_PERSIST"])
def test_fallback_paths_in_subprocess(gpu, env):
    """The two-plane ticket stop test (used when the third plane cannot be
    allocated) and ordinary launches (no PDL) give the same results."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, **{env: "1"})
    r = subprocess.run([sys.executable, "-c", _SUBPROC % root], env=e, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("rows,cols", [(1, 1), (3, 5), (31, 33), (64, 64), (100, 120), (90, 130)])
def test_small_kernel_iterate_and_solve(gpu, orc, dtype, rows, cols):
    """K5 (whole grid in one CTA's shared memory, every iteration and the stop
    test in one launch) on odd, ragged and degenerate shapes."""
    init = _field(rows, cols, seed=rows * 7 + cols, dtype=dtype)
    ref, rep = _oracle_iterate(orc, init, dtype, 1.6, 13, measure_last=True)
    with gpu.Grid.create(init, dtype=dtype) as g:
        g.set_kernel("small")
        d = g.iterate(1.6, 13, want_delta=True)
        assert np.array_equal(g.download(), ref) and d == rep.max_change
        u = orc.to_storage(ref, dtype)
        rr = orc.solve(u, 1.9, 1e-5, 600, 3)
        r = g.solve(1.9, 1e-5, 600, 3)
        assert (r.converged, r.iters, r.max_change) == (rr.status == 0, rr.iters, rr.max_change)
        assert np.array_equal(g.download(), u.astype(np.float64))
