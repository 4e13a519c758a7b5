"""Temporal depth T = 5, 6 (SOR_KERNEL_TEMPORAL, single-slab handles, the
skew-2 kernel only): bitwise against the oracle (`-m gpu`) for iterate with
remainder passes, solve with every-iteration checks (probe / high-word /
exact re-run paths) and cadence K > 1; rejected on multi-slab handles and
for Jacobi."""
import numpy as np
import pytest

import sor_inputs as SI

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu(sor):
    import torch
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return sor


@pytest.mark.parametrize("T", [5, 6])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("rows,cols", [(1, 1), (7, 9), (31, 33), (65, 127), (130, 257), (300, 517), (613, 1029)])
def test_deep_t_iterate_bitwise(gpu, orc, T, dtype, rows, cols):
    init = SI.random_field(rows, cols, seed=rows + cols, lo=-50.0, hi=100.0)
    for iters in (1, T + 2, 3 * T):
        ref = orc.to_storage(init, dtype)
        rep = orc.iterate(ref, 1.93, iters, measure_last=True)
        with gpu.Grid.create(init, dtype=dtype) as g:
            g.set_kernel("temporal", T)
            d = g.iterate(1.93, iters, want_delta=True)
            out = g.download()
        assert np.array_equal(out, ref.astype(np.float64)), (rows, cols, T, dtype, iters)
        assert d == rep.max_change


@pytest.mark.parametrize("T", [5, 6])
@pytest.mark.parametrize("K", [1, 3])
def test_deep_t_solve_exact(gpu, orc, T, K):
    init = SI.random_edges(150, 203, seed=T * 10 + K)
    ref = init.copy()
    orc.iterate(ref, 1.9, 40)
    rr = orc.solve(ref, 1.9, 1e-7, 4000, K)
    with gpu.Grid.create(init) as g:
        g.set_kernel("temporal", T)
        g.iterate(1.9, 40)
        r = g.solve(1.9, 1e-7, 4000, K)
        out = g.download()
    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
    assert np.array_equal(out, ref)


def test_deep_t_c1(gpu, orc):
    cfg = SI.config("C1")
    ref = cfg.init()
    rr = orc.solve(ref, cfg.omega, cfg.tol, cfg.maxit, 1)
    for T in (5, 6):
        with gpu.Grid.create(cfg.init()) as g:
            g.set_kernel("temporal", T)
            r = g.solve(cfg.omega, cfg.tol, cfg.maxit, 1)
            out = g.download()
        assert (r.converged, r.iters, r.max_change) == (True, rr.iters, rr.max_change)
        assert np.array_equal(out, ref)


def test_deep_t_rejected_where_unsupported(gpu):
    init = SI.random_edges(64, 64, seed=1)
    with gpu.Grid.create_virtual(init, 2) as g:
        with pytest.raises(gpu.SorError):
            g.set_kernel("temporal", 5)
    with gpu.Grid.create(init) as g:
        g.set_kernel("temporal", 6)
        with pytest.raises(gpu.SorError):
            g.jacobi(4)
        with pytest.raises(gpu.SorError):
            g.set_kernel("temporal", 7)
