"""NEXT-3: 3-D red-black SOR on the GPU (sor3d_* ABI) vs the oracle (`-m gpu`),
bitwise: grids, iteration counts, reported max-changes."""
import numpy as np
import pytest

import sor_inputs as SI

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1, 1), (2, 3, 5), (7, 6, 9), (16, 16, 16), (9, 40, 300), (33, 17, 130)]


@pytest.fixture(scope="module")
def gpu(sor):
    import torch
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return sor


@pytest.mark.parametrize("kernel", ["fused", "natural"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("shape", SHAPES)
def test_sor3d_iterate_bitwise(gpu, orc, kernel, dtype, shape):
    nz, ny, nx = shape
    init = SI.random_field3d(nz, ny, nx, seed=nz * 100 + ny * 10 + nx, lo=-50.0, hi=100.0)
    ref = init.copy() if dtype == "f64" else init.astype(np.float32)
    rep = orc.sor3d_iterate(ref, 1.7, 9, measure_last=True)
    with gpu.Grid3D(init, dtype=dtype) as g:
        g.set_kernel(kernel)
        d = g.iterate(1.7, 9, want_delta=True)
        out = g.download()
    assert np.array_equal(out, ref.astype(np.float64))
    assert d == rep.max_change


@pytest.mark.parametrize("kernel", ["fused", "natural"])
@pytest.mark.parametrize("K", [1, 5])
def test_sor3d_solve_exact(gpu, orc, kernel, K):
    init = SI.random_shell3d(20, 24, 28, seed=K)
    ref = init.copy()
    rr = orc.sor3d_solve(ref, 1.8, 1e-6, 5000, K)
    rr2 = orc.sor3d_solve(ref, 1.8, 1e-30, 13, 1)
    with gpu.Grid3D(init) as g:
        g.set_kernel(kernel)
        r = g.solve(1.8, 1e-6, 5000, K)
        r2 = g.solve(1.8, 1e-30, 13, 1)
        out = g.download()
    assert (r.converged, r.iters, r.max_change) == (True, rr.iters, rr.max_change) and rr.converged
    assert (r2.converged, r2.iters, r2.max_change) == (False, 13, rr2.max_change)
    assert np.array_equal(out, ref)


def test_sor3d_errors(gpu):
    init = SI.top_hot3d(4, 4, 4, 1.0)
    with gpu.Grid3D(init) as g:
        with pytest.raises(gpu.SorError):
            g.iterate(2.0, 1)
        with pytest.raises(gpu.SorError):
            g.solve(1.5, 1e-3, 10, 11)
        g.iterate(1.5, 2)
    bad = init.copy()
    bad[2, 2, 2] = np.nan
    with pytest.raises(gpu.SorError):
        gpu.Grid3D(bad)


@pytest.mark.parametrize("seed", [41])
def test_sor3d_random_call_sequences(gpu, orc, seed):
    """Random iterate / solve sequences on random 3-D shapes, both kernels and
    dtypes, against the oracle (bitwise): plane swaps after early exits, the
    stop test at every cadence, continuation across calls."""
    import random
    rng = random.Random(seed)
    for case in range(150):
        nz, ny, nx = rng.randint(1, 24), rng.randint(1, 30), rng.randint(1, 140)
        kernel = rng.choice(["fused", "natural"])
        dtype = rng.choice(["f64", "f64", "f32"])
        init = SI.random_field3d(nz, ny, nx, seed=rng.randint(0, 10**6), lo=-50.0, hi=100.0)
        ref = init.copy() if dtype == "f64" else init.astype(np.float32)
        with gpu.Grid3D(init, dtype=dtype) as g:
            g.set_kernel(kernel)
            for _ in range(rng.randint(1, 4)):
                omega = rng.choice([1.0, 1.5, 1.8, 0.5])
                if rng.random() < 0.4:
                    k = rng.randint(0, 25)
                    g.iterate(omega, k)
                    orc.sor3d_iterate(ref, omega, k)
                else:
                    tol = 10 ** rng.uniform(-8, -1)
                    K = rng.choice([1, 2, 5])
                    maxit = rng.choice([500, 60, 7])
                    if K > maxit:
                        K = 1
                    r = g.solve(omega, tol, maxit, K)
                    rr = orc.sor3d_solve(ref, omega, tol, maxit, K)
                    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change), \
                        (case, nz, ny, nx, kernel, dtype)
            assert np.array_equal(g.download(), ref.astype(np.float64)), (case, nz, ny, nx, kernel, dtype)


@pytest.mark.parametrize("kernel", ["fused", "natural"])
@pytest.mark.parametrize("dtype,scale", [("f64", 1e-305), ("f64", 1.0), ("f32", 1e-36)])
def test_sor3d_tiny_values_and_chunks(gpu, orc, kernel, dtype, scale):
    """Reading N3-2's integer path for tiny quotients: a shell scaled into the
    subnormal range (and a zero interior) makes the s/6 of the diffusion front
    tiny or subnormal; shapes give several (y, x) tiles, ragged tiles and
    several z chunks of the fused kernel.  Bitwise against the oracle."""
    init = SI.random_shell3d(37, 45, 97, seed=5) * scale
    init[1:-1, 1:-1, 1:-1] = SI.random_field3d(37, 45, 97, seed=6, lo=0.0, hi=1.0)[1:-1, 1:-1, 1:-1] * scale * 1e-3
    ref = init.copy() if dtype == "f64" else init.astype(np.float32)
    rep = orc.sor3d_iterate(ref, 1.85, 23, measure_last=True)
    with gpu.Grid3D(init, dtype=dtype) as g:
        g.set_kernel(kernel)
        d = g.iterate(1.85, 23, want_delta=True)
        out = g.download()
    assert np.array_equal(out, ref.astype(np.float64))
    assert d == rep.max_change
