"""NEXT-4: multi-colour SOR and block red-black SOR (DESIGN.md readings
N4-1 / N4-2) on the GPU through the C ABI vs the oracle (`-m gpu`), bitwise:
grids, iteration counts, reported max-changes."""
import numpy as np
import pytest

import sor_inputs as SI

pytestmark = pytest.mark.gpu

MC = [(1, 1, 2), (1, 1, 4), (1, 2, 3), (3, 1, 4), (2, 3, 5), (1, -1, 3), (5, 2, 8), (1, 1, 8)]
BLOCKS = [1, 2, 3, 5, 8, 13, 16, 32]
SIZES = [(1, 1), (1, 9), (9, 1), (5, 7), (31, 33), (64, 64), (97, 130), (130, 257), (300, 517)]


@pytest.fixture(scope="module")
def gpu(sor):
    import torch
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return sor


def _mc_ref(orc, init, dtype, mc, iters, measure_last=True):
    ref = orc.to_storage(init, dtype)
    rep = orc.multicolor_iterate(ref, 1.63, iters, *mc, measure_last=measure_last)
    return ref, rep


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("mc", MC)
@pytest.mark.parametrize("rows,cols", SIZES)
def test_multicolor_iterate_bitwise(gpu, orc, dtype, mc, rows, cols):
    init = SI.random_field(rows, cols, seed=rows * 13 + cols + mc[2], lo=-50.0, hi=100.0)
    ref, rep = _mc_ref(orc, init, dtype, mc, 5)
    with gpu.Grid.create(init, dtype=dtype) as g:
        d = g.variant_iterate(gpu.Variant.multicolor(*mc), 1.63, 5, want_delta=True)
        out = g.download()
        assert g.stats["half_sweeps"] == 5 * mc[2]
    assert np.array_equal(out, ref.astype(np.float64))
    assert d == rep.max_change


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("B", BLOCKS)
@pytest.mark.parametrize("rows,cols", SIZES)
def test_block_iterate_bitwise(gpu, orc, dtype, B, rows, cols):
    init = SI.random_field(rows, cols, seed=rows * 17 + cols + B, lo=-50.0, hi=100.0)
    ref = orc.to_storage(init, dtype)
    rep = orc.block_iterate(ref, 1.71, 4, B, measure_last=True)
    with gpu.Grid.create(init, dtype=dtype) as g:
        d = g.variant_iterate(gpu.Variant.blocks(B), 1.71, 4, want_delta=True)
        out = g.download()
        assert g.stats["half_sweeps"] == 8
    assert np.array_equal(out, ref.astype(np.float64))
    assert d == rep.max_change


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_two_colours_and_block_one_equal_red_black_kernels(gpu, orc, dtype):
    init = SI.random_edges(200, 333, seed=4)
    outs = []
    for call in (lambda g: g.iterate(1.9, 9), lambda g: g.variant_iterate(gpu.Variant.multicolor(1, 1, 2), 1.9, 9),
                 lambda g: g.variant_iterate(gpu.Variant.blocks(1), 1.9, 9)):
        with gpu.Grid.create(init, dtype=dtype) as g:
            g.set_kernel("temporal", 3)
            call(g)
            outs.append(g.download())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("variant", [("mc", (1, 1, 4)), ("mc", (1, 2, 3)), ("block", 4), ("block", 7)])
@pytest.mark.parametrize("K", [1, 3])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_variant_solve_exact(gpu, orc, variant, K, dtype):
    init = SI.random_edges(48, 61, seed=K + 5)
    ref = orc.to_storage(init, dtype)
    tol = 1e-6 if dtype == "f64" else 1e-3
    if variant[0] == "mc":
        v = gpu.Variant.multicolor(*variant[1])
        rep = orc.multicolor_solve(ref, 1.8, tol, 20000, K, *variant[1])
    else:
        v = gpu.Variant.blocks(variant[1])
        rep = orc.block_solve(ref, 1.8, tol, 20000, variant[1], K)
    assert rep.converged
    with gpu.Grid.create(init, dtype=dtype) as g:
        r = g.variant_solve(v, 1.8, tol, 20000, K)
        out = g.download()
    assert r.converged and r.iters == rep.iters and r.max_change == rep.max_change
    assert np.array_equal(out, ref.astype(np.float64))


def test_variant_solve_not_converged_and_continuation(gpu, orc):
    init = SI.random_edges(40, 40, seed=9)
    ref = init.copy()
    r1 = orc.block_solve(ref, 1.5, 1e-12, 30, 3, 4)
    orc.multicolor_iterate(ref, 1.5, 7, 1, 2, 3)
    with gpu.Grid.create(init) as g:
        r = g.variant_solve(gpu.Variant.blocks(3), 1.5, 1e-12, 30, 4)
        assert not r.converged and r.iters == 30 and r.max_change == r1.max_change
        g.variant_iterate(gpu.Variant.multicolor(1, 2, 3), 1.5, 7)
        out = g.download()
    assert np.array_equal(out, ref)


def test_variant_after_deferred_solve_and_mixing(gpu, orc):
    """Variants share the handle's planes with the SOR kernels (incl. the third
    plane of the deferred stop test)."""
    init = SI.random_edges(257, 300, seed=3)
    ref = init.copy()
    rr = orc.solve(ref, 1.9, 1e-3, 5000, 1)
    orc.block_iterate(ref, 1.9, 5, 2)
    orc.iterate(ref, 1.9, 6)
    orc.multicolor_iterate(ref, 1.9, 3, 1, 1, 4)
    with gpu.Grid.create(init) as g:
        g.set_kernel("temporal", 4)
        r = g.solve(1.9, 1e-3, 5000, 1)
        assert r.iters == rr.iters
        g.variant_iterate(gpu.Variant.blocks(2), 1.9, 5)
        g.iterate(1.9, 6)
        g.variant_iterate(gpu.Variant.multicolor(1, 1, 4), 1.9, 3)
        out = g.download()
    assert np.array_equal(out, ref)


def test_variant_full_size_bitwise(gpu, orc):
    """BASELINE configs[2] size (4096^2, the bench workload of the NEXT-4 lines),
    whole grid vs the oracle after 3 iterations of each variant."""
    cfg = SI.config("C3")
    init = cfg.init()
    for v, f in ((gpu.Variant.multicolor(1, 1, 4), lambda u: orc.multicolor_iterate(u, cfg.omega, 3, 1, 1, 4,
                                                                                    measure_last=True)),
                 (gpu.Variant.blocks(8), lambda u: orc.block_iterate(u, cfg.omega, 3, 8, measure_last=True))):
        ref = init.copy()
        rep = f(ref)
        with gpu.Grid.create(init) as g:
            d = g.variant_iterate(v, cfg.omega, 3, want_delta=True)
            out = g.download()
        assert np.array_equal(out, ref) and d == rep.max_change


def test_variant_invalid_and_unsupported(gpu):
    init = SI.north_hot(20, 20, 1.0)
    with gpu.Grid.create(init) as g:
        for v, code in ((gpu.Variant.multicolor(2, 1, 2), gpu.SOR_E_INVAL),
                        (gpu.Variant.multicolor(1, 1, 9), gpu.SOR_E_UNSUPPORTED),
                        (gpu.Variant.multicolor(1, 1, 1), gpu.SOR_E_UNSUPPORTED),
                        (gpu.Variant.blocks(0), gpu.SOR_E_UNSUPPORTED),
                        (gpu.Variant.blocks(33), gpu.SOR_E_UNSUPPORTED),
                        (gpu.Variant(7, 0, 0, 0, 0), gpu.SOR_E_INVAL)):
            with pytest.raises(gpu.SorError) as e:
                g.variant_iterate(v, 1.5, 1)
            assert e.value.code == code
        with pytest.raises(gpu.SorError):
            g.variant_iterate(gpu.Variant.blocks(2), 2.0, 1)
        assert g.variant_iterate(gpu.Variant.blocks(2), 1.5, 0, want_delta=True) == 0.0
        g.iterate(1.5, 2)  # still usable
    with gpu.Grid.create_virtual(init, 2) as g:
        with pytest.raises(gpu.SorError) as e:
            g.variant_iterate(gpu.Variant.blocks(2), 1.5, 1)
        assert e.value.code == gpu.SOR_E_UNSUPPORTED
