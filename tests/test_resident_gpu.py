"""K7 (SOR_KERNEL_RESIDENT, resident.cuh): the grid register-resident across
the SMs, compared with the oracle bitwise (`-m gpu`).

Multi-CTA iterate: 2-D blocks of the interior, one per SM, each window = the
block + a 2T ring; blocks exchange only their 2T-deep frames with the 8
neighbouring blocks between passes (flags, no grid barrier).  The shapes below
give 2..148 blocks, blocks as thin as 2T rows, ragged block sizes, odd/even
origins, and iteration counts that leave a short last pass.  Single CTA
(grids of <= 126 columns): iterate and solve with the device-side stop test.
Grids that fit neither run as SOR_KERNEL_TEMPORAL (fallback, also checked).
"""
import numpy as np
import pytest

import sor_inputs as SI

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu(sor):
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    torch.cuda.set_device(0)
    return sor


def _field(rows, cols, seed):
    return SI.random_field(rows, cols, seed=seed, lo=-50.0, hi=100.0)


MULTI = [(16, 130), (64, 64), (97, 250), (128, 128), (300, 517), (613, 1029), (1024, 1024), (1000, 1030),
         (1187, 1201)]


@pytest.mark.parametrize("T", [1, 2, 3, 4])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("rows,cols", MULTI)
def test_resident_iterate_bitwise(gpu, orc, T, dtype, rows, cols):
    init = _field(rows, cols, seed=rows * 7 + cols)
    for iters in (1, 2 * T + 1 if T > 1 else 5, 13):
        ref = orc.to_storage(init, dtype)
        rep = orc.iterate(ref, 1.93, iters, measure_last=True)
        with gpu.Grid.create(init, dtype=dtype) as g:
            g.set_kernel("resident", T)
            d = g.iterate(1.93, iters, want_delta=True)
            out = g.download()
            st = g.stats
        assert np.array_equal(out, ref.astype(np.float64)), (rows, cols, T, dtype, iters)
        assert d == rep.max_change
        assert st["half_sweeps"] == 2 * iters


@pytest.mark.parametrize("T", [2, 3, 4])
def test_resident_one_launch(gpu, orc, T):
    """C2-sized grid: the whole iterate call is one launch (multi-CTA form)."""
    init = _field(1024, 1024, seed=T)
    with gpu.Grid.create(init) as g:
        g.set_kernel("resident", T)
        g.iterate(1.9, 40)
        st = g.stats
    assert st["kernel_launches"] == 1


@pytest.mark.parametrize("T", [1, 3, 4])
def test_resident_continuation_and_reset(gpu, orc, T):
    """Consecutive launches on one handle (flag epochs, plane alternation with
    odd and even pass counts), omega changes, zero-iteration calls, reset."""
    init = _field(613, 1029, seed=11)
    ref = init.copy()
    with gpu.Grid.create(init) as g:
        g.set_kernel("resident", T)
        for omega, n in ((1.5, 3), (1.99, 7), (1.2, 0), (1.93, 1), (0.376, 12), (1.7, 5)):
            orc.iterate(ref, omega, n)
            g.iterate(omega, n)
        assert np.array_equal(g.download(), ref)
        g.reset(init)
        ref = init.copy()
        orc.iterate(ref, 1.8, 9)
        g.iterate(1.8, 9)
        assert np.array_equal(g.download(), ref)


def test_resident_mixed_with_wave_kernels(gpu, orc):
    """Kernel switches on one handle: K7 iterate, K4 iterate / solve, K7 again."""
    init = _field(300, 517, seed=3)
    ref = init.copy()
    with gpu.Grid.create(init) as g:
        g.set_kernel("resident", 3)
        g.iterate(1.9, 10)
        orc.iterate(ref, 1.9, 10)
        g.set_kernel("temporal", 4)
        g.iterate(1.9, 6)
        orc.iterate(ref, 1.9, 6)
        r = g.solve(1.9, 1e-3, 500, 1)
        rr = orc.solve(ref, 1.9, 1e-3, 500, 1)
        assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
        g.set_kernel("resident", 2)
        g.iterate(1.95, 7)
        orc.iterate(ref, 1.95, 7)
        # solve on a grid too wide for one CTA runs as TEMPORAL depth T
        r = g.solve(1.95, 1e-4, 300, 1)
        rr = orc.solve(ref, 1.95, 1e-4, 300, 1)
        assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
        assert np.array_equal(g.download(), ref)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("rows,cols", [(1, 1), (1, 126), (94, 126), (64, 64), (30, 90), (90, 3)])
@pytest.mark.parametrize("K", [1, 4])
def test_resident_single_cta_solve(gpu, orc, dtype, rows, cols, K):
    """One-CTA form (window = whole grid): solve with the stop test on the
    device, then maxit exhaustion; and iterate with the last max-change."""
    init = SI.random_edges(rows, cols, seed=rows + 3 * cols)
    ref = orc.to_storage(init, dtype)
    rr = orc.solve(ref, 1.8, 1e-6, 3000, K)
    with gpu.Grid.create(init, dtype=dtype) as g:
        g.set_kernel("resident", 1)
        r = g.solve(1.8, 1e-6, 3000, K)
        assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
        assert g.stats["kernel_launches"] == 1
        assert np.array_equal(g.download(), ref.astype(np.float64))
        rr2 = orc.solve(ref, 1.9, 1e-30, 17, K)
        r2 = g.solve(1.9, 1e-30, 17, K)
        assert (r2.converged, r2.iters, r2.max_change) == (rr2.converged, rr2.iters, rr2.max_change) == \
            (False, 17, rr2.max_change)
        rep = orc.iterate(ref, 1.3, 6, measure_last=True)
        d = g.iterate(1.3, 6, want_delta=True)
        assert d == rep.max_change
        assert np.array_equal(g.download(), ref.astype(np.float64))


def test_resident_fallback_large(gpu, orc):
    """Too large for one block per SM: iterate runs as TEMPORAL (bitwise)."""
    init = _field(1500, 2100, seed=9)
    ref = init.copy()
    rep = orc.iterate(ref, 1.9, 9, measure_last=True)
    with gpu.Grid.create(init) as g:
        g.set_kernel("resident", 4)
        d = g.iterate(1.9, 9, want_delta=True)
        assert g.stats["kernel_launches"] > 1
        out = g.download()
    assert np.array_equal(out, ref) and d == rep.max_change


def test_resident_c1(gpu, orc):
    """BJ configs[0] on the one-CTA form: 1785 iterations, bitwise grid."""
    cfg = SI.config("C1")
    ref = cfg.init()
    rr = orc.solve(ref, cfg.omega, cfg.tol, cfg.maxit, 1)
    with gpu.Grid.create(cfg.init()) as g:
        g.set_kernel("resident", 1)
        r = g.solve(cfg.omega, cfg.tol, cfg.maxit, 1)
        out = g.download()
    assert (r.converged, r.iters, r.max_change) == (True, rr.iters, rr.max_change) == (True, 1785, rr.max_change)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("nslabs", [2, 3])
def test_resident_on_virtual_slabs_falls_back(gpu, orc, nslabs):
    """SOR_KERNEL_RESIDENT on a multi-slab handle runs the slab path at depth T
    (K7 needs one slab): bitwise, iterate and solve."""
    init = _field(203, 150, seed=nslabs)
    ref = init.copy()
    rep = orc.iterate(ref, 1.9, 11, measure_last=True)
    with gpu.Grid.create_virtual(init, nslabs) as g:
        g.set_kernel("resident", 3)
        d = g.iterate(1.9, 11, want_delta=True)
        assert np.array_equal(g.download(), ref) and d == rep.max_change
        r = g.solve(1.9, 1e-4, 400, 1)
        rr = orc.solve(ref, 1.9, 1e-4, 400, 1)
        assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
        assert np.array_equal(g.download(), ref)


def test_resident_on_external_stream(gpu, orc):
    """K7 launches go to the handle's stream (an external torch stream here),
    ordered with the caller's work on it."""
    import torch
    init = _field(613, 1029, seed=21)
    ref = init.copy()
    orc.iterate(ref, 1.8, 9)
    s = torch.cuda.Stream()
    with gpu.Grid.create(init) as g:
        g.set_kernel("resident", 3)
        g.set_stream(s.cuda_stream)
        g.iterate(1.8, 9)
        s.synchronize()
        out = g.download()
    assert np.array_equal(out, ref)
