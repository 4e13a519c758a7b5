"""NEXT-2: Jacobi on the GPU through the C ABI vs the oracle
(`-m gpu`), bitwise: grids, iteration counts, reported max-changes."""
import numpy as np
import pytest

import sor_inputs as SI

pytestmark = pytest.mark.gpu

KERNELS = [("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4)]
SIZES = [(1, 1), (3, 5), (8, 8), (31, 33), (64, 64), (130, 257), (257, 130), (300, 517)]


@pytest.fixture(scope="module")
def gpu(sor):
    import torch
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return sor


@pytest.mark.parametrize("kernel,T", KERNELS)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("rows,cols", SIZES)
def test_jacobi_iterate_bitwise(gpu, orc, kernel, T, dtype, rows, cols):
    init = SI.random_field(rows, cols, seed=rows * 7 + cols, lo=-50.0, hi=100.0)
    ref = orc.to_storage(init, dtype)
    rep = orc.jacobi_iterate(ref, 7, measure_last=True)
    with gpu.Grid.create(init, dtype=dtype) as g:
        g.set_kernel(kernel, T)
        d = g.jacobi(7, want_delta=True)
        out = g.download()
    assert np.array_equal(out, ref.astype(np.float64))
    assert d == rep.max_change


@pytest.mark.parametrize("kernel,T", KERNELS)
@pytest.mark.parametrize("K", [1, 4])
def test_jacobi_solve_and_mixing_with_sor(gpu, orc, kernel, T, K):
    init = SI.random_edges(70, 95, seed=K + T)
    ref = init.copy()
    orc.iterate(ref, 1.7, 5)                          # SOR first, then Jacobi on the same handle
    rr = orc.jacobi_solve(ref, 1e-3, 3000, K)
    rr2 = orc.jacobi_solve(ref, 1e-30, 30, K)         # maxit reached
    with gpu.Grid.create(init) as g:
        g.set_kernel(kernel, T)
        g.iterate(1.7, 5)
        r = g.jacobi_solve(1e-3, 3000, K)
        r2 = g.jacobi_solve(1e-30, 30, K)
        st = g.stats
        out = g.download()
    assert st["half_sweeps"] == 30          # one Jacobi sweep per iteration
    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change)
    assert (r2.converged, r2.iters, r2.max_change) == (False, 30, rr2.max_change)
    assert np.array_equal(out, ref)


def test_jacobi_converges_to_the_sor_fixed_point(gpu):
    """converged Jacobi and converged SOR agree within ~10 tol."""
    init = SI.random_edges(40, 40, seed=2)
    with gpu.Grid.create(init) as g:
        g.set_kernel("temporal", 4)
        r = g.solve(1.85, 1e-12, 100000, 1)
        sor = g.download()
    with gpu.Grid.create(init) as g:
        g.set_kernel("temporal", 4)
        rj = g.jacobi_solve(1e-12, 200000, 1)
        jac = g.download()
    assert r.converged and rj.converged
    assert np.abs(sor - jac).max() < 1e-8


def test_jacobi_rejects_unsupported_kernels(gpu):
    init = SI.north_hot(10, 10, 1.0)
    with gpu.Grid.create(init) as g:
        g.set_kernel("natural")
        with pytest.raises(gpu.SorError) as e:
            g.jacobi(3)
        assert e.value.code == gpu.SOR_E_UNSUPPORTED
        g.set_kernel("fused")
        with pytest.raises(gpu.SorError):
            g.jacobi(-1)
        with pytest.raises(gpu.SorError):
            g.jacobi_solve(0.0, 10)
