"""Pins for the NEXT-4 oracle (oracle/sor_oracle.c `orc_variant_run_*`).

The paper names multi-colour SOR and block-parallel SOR beside red-black SOR
[§3.1, P:147] without defining them; DESIGN.md §3 readings N4-1 (multi-colour:
colour (ca*i + cb*j) mod nc, phases 0..nc-1) and N4-2 (block red-black: a
chessboard of B x B blocks, red first, natural order inside a block) are the
definitions.  Every update is Eq. 1 [P:97-100] in the canonical order.

The oracle is pinned against references that share nothing with it:
  * special cases that reduce to methods pinned elsewhere: (1, 1, 2) and B = 1
    are the paper's red-black SOR [P:149, P:198] (and the naive guarded
    Code-1 sweep [P:158-169]); one colour per cell in lexicographic order, and
    B >= max(rows, cols), are natural-order SOR (a plain sequential sweep);
  * brute force with a different loop structure: a colour phase as ONE
    simultaneous (Jacobi-style) update of all its cells, and a block phase as
    B*B simultaneous steps over all blocks of the colour (position t of every
    block at step t) — both equal the sequential definition only because the
    colouring is valid, so a wrong colouring, order or neighbour fails;
  * the fixed point is the dense direct solution of the 5-point system, and a
    discrete-harmonic grid is left unchanged;
  * fp32: the same brute force in numpy float32 (per-op rounding in float).
"""
import numpy as np
import pytest

import sor_inputs as SI


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build_oracle()
    return oracle


def _upd(u, i, j, w, dt):
    """Eq. 1, canonical order, every op in dt (numpy scalar arithmetic)."""
    s = (u[i - 1, j] + u[i + 1, j]) + (u[i, j - 1] + u[i, j + 1])
    a = dt(0.25) * s
    return u[i, j] + w * (a - u[i, j])


def _natural_sweep(u, omega, iters):
    """Natural-order (lexicographic) SOR: a plain sequential sweep."""
    dt = u.dtype.type
    w = dt(omega)
    rows, cols = u.shape[0] - 2, u.shape[1] - 2
    for _ in range(iters):
        for i in range(1, rows + 1):
            for j in range(1, cols + 1):
                u[i, j] = _upd(u, i, j, w, dt)


def _mc_simultaneous(u, omega, iters, ca, cb, nc):
    """Each colour phase as one simultaneous update (new values from a copy)."""
    dt = u.dtype.type
    w = dt(omega)
    rows, cols = u.shape[0] - 2, u.shape[1] - 2
    for _ in range(iters):
        for p in range(nc):
            old = u.copy()
            for i in range(1, rows + 1):
                for j in range(1, cols + 1):
                    if (ca * i + cb * j) % nc == p:
                        u[i, j] = _upd(old, i, j, w, dt)


def _block_simultaneous(u, omega, iters, B):
    """Block red-black: B*B steps per colour; step t updates position
    (t // B, t % B) of every block of the colour at once (from a copy)."""
    dt = u.dtype.type
    w = dt(omega)
    rows, cols = u.shape[0] - 2, u.shape[1] - 2
    nbi, nbj = -(-rows // B), -(-cols // B)
    for _ in range(iters):
        for c in (0, 1):
            for t in range(B * B):
                old = u.copy()
                di, dj = divmod(t, B)
                for bi in range(nbi):
                    for bj in range(nbj):
                        if (bi + bj) % 2 != c:
                            continue
                        i, j = 1 + bi * B + di, 1 + bj * B + dj
                        if i <= rows and j <= cols:
                            u[i, j] = _upd(old, i, j, w, dt)


def _redblack_naive(u, omega, iters):
    """The paper's Code 1 guarded sweep: red phase, black phase."""
    dt = u.dtype.type
    w = dt(omega)
    rows, cols = u.shape[0] - 2, u.shape[1] - 2
    for _ in range(iters):
        for c in (0, 1):
            for i in range(1, rows + 1):
                for j in range(1, cols + 1):
                    if (i + j) % 2 == c:
                        u[i, j] = _upd(u, i, j, w, dt)


DTYPES = [np.float64, np.float32]


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("rows,cols", [(1, 1), (3, 8), (7, 5), (6, 6)])
def test_mc_two_colours_is_red_black(orc, dt, rows, cols):
    u = SI.random_field(rows, cols, seed=rows * 31 + cols).astype(dt)
    v, x = u.copy(), u.copy()
    r = orc.multicolor_iterate(u, 1.37, 5, 1, 1, 2, measure_last=True)
    _redblack_naive(v, 1.37, 5)
    assert np.array_equal(u, v)
    rr = orc.iterate(x, 1.37, 5, measure_last=True)
    assert np.array_equal(u, x) and r.max_change == rr.max_change
    assert r.half_sweeps == 10


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("ca,cb,nc", [(1, 1, 4), (1, 2, 3), (3, 1, 4), (2, 3, 5), (1, -1, 3), (5, 2, 8)])
@pytest.mark.parametrize("rows,cols", [(4, 6), (7, 5)])
def test_mc_equals_simultaneous_phases(orc, dt, ca, cb, nc, rows, cols):
    u = SI.random_field(rows, cols, seed=nc * 100 + rows).astype(dt)
    v = u.copy()
    orc.multicolor_iterate(u, 1.61, 3, ca, cb, nc)
    _mc_simultaneous(v, 1.61, 3, ca, cb, nc)
    assert np.array_equal(u, v)


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("rows,cols", [(1, 6), (4, 5), (6, 3)])
def test_mc_one_colour_per_cell_is_natural_order(orc, dt, rows, cols):
    u = SI.random_field(rows, cols, seed=7 + rows).astype(dt)
    v = u.copy()
    nc = cols * rows + cols + 1          # ca*i + j is distinct and lexicographic
    r = orc.multicolor_iterate(u, 1.2, 3, cols, 1, nc)
    _natural_sweep(v, 1.2, 3)
    assert np.array_equal(u, v)
    assert r.half_sweeps == 3 * nc


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("rows,cols", [(1, 1), (5, 8), (9, 4)])
def test_block_one_is_red_black(orc, dt, rows, cols):
    u = SI.random_field(rows, cols, seed=rows + 3 * cols).astype(dt)
    v = u.copy()
    r = orc.block_iterate(u, 1.45, 4, 1, measure_last=True)
    rr = orc.iterate(v, 1.45, 4, measure_last=True)
    assert np.array_equal(u, v) and r.max_change == rr.max_change


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("rows,cols,B", [(5, 7, 7), (6, 3, 6), (4, 4, 9)])
def test_block_whole_grid_is_natural_order(orc, dt, rows, cols, B):
    u = SI.random_field(rows, cols, seed=B).astype(dt)
    v = u.copy()
    orc.block_iterate(u, 1.3, 3, B)
    _natural_sweep(v, 1.3, 3)
    assert np.array_equal(u, v)


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("rows,cols,B", [(6, 6, 2), (7, 9, 3), (10, 5, 4), (5, 11, 2), (8, 8, 3)])
def test_block_equals_simultaneous_positions(orc, dt, rows, cols, B):
    u = SI.random_field(rows, cols, seed=rows * cols + B).astype(dt)
    v = u.copy()
    orc.block_iterate(u, 1.7, 3, B)
    _block_simultaneous(v, 1.7, 3, B)
    assert np.array_equal(u, v)


@pytest.mark.parametrize("variant", [("mc", 1, 1, 4), ("mc", 1, 2, 3), ("block", 3), ("block", 4)])
def test_variants_converge_to_dense_solution(orc, variant):
    u = SI.random_edges(9, 11, seed=5)
    ref = u.copy()
    orc.dense_solve(ref)
    if variant[0] == "mc":
        r = orc.multicolor_solve(u, 1.5, 1e-13, 20000, 1, *variant[1:])
    else:
        r = orc.block_solve(u, 1.5, 1e-13, 20000, variant[1])
    assert r.converged
    assert np.max(np.abs(u - ref)) < 1e-10 * np.max(np.abs(ref))


@pytest.mark.parametrize("variant", [("mc", 1, 1, 4), ("mc", 2, 1, 3), ("block", 2), ("block", 5)])
def test_variants_keep_discrete_harmonic_grid(orc, variant):
    rows, cols = 8, 10
    i, j = np.meshgrid(np.arange(rows + 2), np.arange(cols + 2), indexing="ij")
    u = (0.5 * i + 0.25 * j + 3.0).astype(np.float64)   # dyadic, linear: exact fixed point
    v = u.copy()
    if variant[0] == "mc":
        r = orc.multicolor_iterate(u, 1.3, 4, *variant[1:], measure_last=True)
    else:
        r = orc.block_iterate(u, 1.3, 4, variant[1], measure_last=True)
    assert np.array_equal(u, v) and r.max_change == 0.0


def test_variant_solve_cadence_and_invalid(orc):
    u = SI.random_edges(12, 12, seed=2)
    r = orc.multicolor_solve(u, 1.6, 1e-6, 5000, 7, 1, 1, 4)
    assert r.converged and r.iters % 7 == 0 and r.checks == r.iters // 7
    assert r.half_sweeps == 4 * r.iters
    r = orc.block_solve(SI.random_edges(12, 12, seed=2), 1.6, 1e-6, 5000, 3, 5)
    assert r.converged and r.iters % 5 == 0 and r.half_sweeps == 2 * r.iters
    for bad in ((2, 1, 2), (1, 4, 4), (1, 1, 1)):
        with pytest.raises(ValueError):
            orc.multicolor_iterate(u, 1.5, 1, *bad)
    with pytest.raises(ValueError):
        orc.block_iterate(u, 1.5, 1, 0)


def test_orders_differ(orc):
    """The orderings are genuinely different iterations (not red-black in disguise)."""
    base = SI.random_field(8, 8, seed=11)
    outs = []
    for f in (lambda u: orc.iterate(u, 1.5, 2), lambda u: orc.multicolor_iterate(u, 1.5, 2, 1, 1, 4),
              lambda u: orc.multicolor_iterate(u, 1.5, 2, 1, 2, 3), lambda u: orc.block_iterate(u, 1.5, 2, 2),
              lambda u: orc.block_iterate(u, 1.5, 2, 3)):
        u = base.copy()
        f(u)
        outs.append(u)
    for a in range(len(outs)):
        for b in range(a + 1, len(outs)):
            assert not np.array_equal(outs[a], outs[b]), (a, b)
