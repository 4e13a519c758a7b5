"""Randomised differential test (`-m gpu`): random sequences of iterate /
solve / reset on random grid shapes, kernels and depths, checked against the
oracle (iteration count, reported max-change, final grid, bitwise).  It
exercises the deferred stop test, speculative passes, exact re-runs and the
programmatic-dependent-launch chain between wave kernels (a missing proxy
fence there showed up as ~1 mismatch per 1000 cases before it was fixed).
Fixed seed; ~200 cases."""
import random

import numpy as np
import pytest

import sor_inputs as SI

pytestmark = pytest.mark.gpu

KERNELS = [("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4), ("natural", 1),
           ("resident", 2), ("resident", 3), ("resident", 4)]


@pytest.mark.parametrize("seed", [11, 12])
def test_random_call_sequences(sor, orc, seed):
    import torch
    assert torch.cuda.is_available()
    rng = random.Random(seed)
    for case in range(100):
        rows, cols = rng.randint(1, 300), rng.randint(1, 520)
        kernel, T = rng.choice(KERNELS)
        dtype = rng.choice(["f64", "f64", "f32"])
        init = SI.random_edges(rows, cols, seed=rng.randint(0, 10**6))
        ref = orc.to_storage(init, dtype)
        with sor.Grid.create(init, dtype=dtype) as g:
            g.set_kernel(kernel, T)
            for _ in range(rng.randint(1, 5)):
                op = rng.random()
                omega = rng.choice([1.0, 1.5, 1.9, 1.97, 0.376])
                if op < 0.3:
                    k = rng.randint(0, 40)
                    g.iterate(omega, k)
                    orc.iterate(ref, omega, k)
                elif op < 0.4:
                    g.reset(init)
                    ref = orc.to_storage(init, dtype)
                else:
                    tol = 10 ** rng.uniform(-9, -2)
                    K = rng.choice([1, 1, 1, 2, 5])
                    maxit = rng.choice([1500, 200, 37])
                    r = g.solve(omega, tol, maxit, K)
                    rr = orc.solve(ref, omega, tol, maxit, K)
                    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change), \
                        (case, rows, cols, kernel, T, dtype)
            assert np.array_equal(g.download(), ref.astype(np.float64)), (case, rows, cols, kernel, T, dtype)


@pytest.mark.parametrize("seed", [31])
def test_random_sor_jacobi_sequences(sor, orc, seed):
    """SOR and Jacobi (NEXT-2) calls interleaved at random on one handle: the
    method switch must leave no deferred decision, plane or tile table of one
    method to the other."""
    import torch
    assert torch.cuda.is_available()
    rng = random.Random(seed)
    for case in range(80):
        rows, cols = rng.randint(1, 300), rng.randint(1, 520)
        kernel, T = rng.choice(KERNELS[:4])          # natural has no Jacobi
        dtype = rng.choice(["f64", "f64", "f32"])
        init = SI.random_edges(rows, cols, seed=rng.randint(0, 10**6))
        ref = orc.to_storage(init, dtype)
        with sor.Grid.create(init, dtype=dtype) as g:
            g.set_kernel(kernel, T)
            for _ in range(rng.randint(2, 6)):
                op = rng.random()
                omega = rng.choice([1.0, 1.5, 1.9, 0.376])
                tol = 10 ** rng.uniform(-8, -2)
                K = rng.choice([1, 1, 2, 5])
                maxit = rng.choice([800, 200, 37])
                if op < 0.2:
                    k = rng.randint(0, 30)
                    g.iterate(omega, k)
                    orc.iterate(ref, omega, k)
                elif op < 0.4:
                    k = rng.randint(0, 30)
                    g.jacobi(k)
                    orc.jacobi_iterate(ref, k)
                elif op < 0.7:
                    r = g.solve(omega, tol, maxit, K)
                    rr = orc.solve(ref, omega, tol, maxit, K)
                    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change), \
                        ("sor", case, rows, cols, kernel, T, dtype)
                else:
                    r = g.jacobi_solve(tol, maxit, K)
                    rr = orc.jacobi_solve(ref, tol, maxit, K)
                    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change), \
                        ("jacobi", case, rows, cols, kernel, T, dtype)
            assert np.array_equal(g.download(), ref.astype(np.float64)), (case, rows, cols, kernel, T, dtype)


DEEP_KERNELS = [("fused", 1), ("temporal", 2), ("temporal", 3), ("temporal", 4), ("temporal", 5), ("temporal", 6),
                ("natural", 1)]


def _draw_variant(rng, sor):
    """A random NEXT-4 variant: (binding struct, oracle iterate, oracle solve)."""
    if rng.random() < 0.5:
        nc = rng.randint(2, 8)
        while True:
            ca, cb = rng.randint(-7, 9), rng.randint(-7, 9)
            if ca % nc and cb % nc:
                break
        return (sor.Variant.multicolor(ca, cb, nc), ("mc", ca, cb, nc))
    B = rng.choice([1, 2, 3, 4, 5, 7, 8, 11, 16, 23, 32])
    return (sor.Variant.blocks(B), ("bp", B))


@pytest.mark.parametrize("seed", [41, 42])
def test_random_variant_and_deep_t_sequences(sor, orc, seed):
    """NEXT-4 variant calls (random colourings and block sizes) interleaved on
    one handle with red-black SOR at every kernel and depth up to T = 6, Jacobi
    calls and resets (tools/fuzz_next4.py, bounded): the variants share the
    handle's planes and the deferred solve's third plane with the SOR kernels."""
    import torch
    assert torch.cuda.is_available()
    rng = random.Random(seed)
    for case in range(70):
        rows = rng.choice([rng.randint(1, 40), rng.randint(1, 330)])
        cols = rng.choice([rng.randint(1, 40), rng.randint(1, 560)])
        kernel, T = rng.choice(DEEP_KERNELS)
        dtype = rng.choice(["f64", "f64", "f32"])
        s0 = rng.randint(0, 10**6)
        init = (SI.random_field(rows, cols, seed=s0, lo=-50.0, hi=100.0) if rng.random() < 0.5
                else SI.random_edges(rows, cols, seed=s0))
        ref = orc.to_storage(init, dtype)
        tag = (case, rows, cols, kernel, T, dtype)
        with sor.Grid.create(init, dtype=dtype) as g:
            g.set_kernel(kernel, T)
            for _ in range(rng.randint(1, 6)):
                op, which = rng.random(), rng.random()
                omega = rng.choice([1.0, 1.5, 1.9, 1.97, 0.376])
                pv, v = _draw_variant(rng, sor) if which < 0.6 else (None, None)
                jac = v is None and kernel != "natural" and T <= 4 and which < 0.7
                if op < 0.4:
                    k = rng.randint(0, 25)
                    if v is not None:
                        d = g.variant_iterate(pv, omega, k, want_delta=True)
                        rr = (orc.multicolor_iterate(ref, omega, k, *v[1:], measure_last=True) if v[0] == "mc"
                              else orc.block_iterate(ref, omega, k, v[1], measure_last=True))
                        assert k == 0 or d == rr.max_change, (tag, v)
                    elif jac:
                        g.jacobi(k)
                        orc.jacobi_iterate(ref, k)
                    else:
                        g.iterate(omega, k)
                        orc.iterate(ref, omega, k)
                elif op < 0.5:
                    g.reset(init)
                    ref = orc.to_storage(init, dtype)
                else:
                    tol = 10 ** rng.uniform(-9, -1)
                    K = rng.choice([1, 1, 1, 2, 5])
                    maxit = rng.choice([800, 200, 37])
                    if v is not None:
                        r = g.variant_solve(pv, omega, tol, maxit, K)
                        rr = (orc.multicolor_solve(ref, omega, tol, maxit, K, *v[1:]) if v[0] == "mc"
                              else orc.block_solve(ref, omega, tol, maxit, v[1], K))
                    elif jac:
                        r = g.jacobi_solve(tol, maxit, K)
                        rr = orc.jacobi_solve(ref, tol, maxit, K)
                    else:
                        r = g.solve(omega, tol, maxit, K)
                        rr = orc.solve(ref, omega, tol, maxit, K)
                    assert (r.converged, r.iters, r.max_change) == (rr.converged, rr.iters, rr.max_change), (tag, v)
            assert np.array_equal(g.download(), ref.astype(np.float64)), tag
