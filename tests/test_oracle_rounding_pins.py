"""Rounding pins for the CPU oracle: every arithmetic operation is rounded to T.

Readings #2-#4 and #17 fix not only WHAT Eq. 1 computes
[§2.1 Eq. 1, P:97-100] but how each operation rounds: the canonical order
s = (N+S)+(W+E); a = 0.25*s; r = a - u; u' = u + w*r, each step rounded to
the storage type T (fp64, or fp32 for C4-f32), no FMA contraction, no wider
intermediates.  The 3-D extension [P:410] divides by 6 with one correctly
rounded division (reading N3-1).  The pins in tests/test_oracle_pins.py fix
the algorithm in fp64; these fix the per-operation rounding, so that a
mutation of the oracle that computes in double and rounds once, that
replaces s/6 by s*(1/6), or that reorders a sum fails here.

Two independent references, neither sharing code with oracle/:
  * exact rational arithmetic (fractions.Fraction) with an explicit
    round-to-nearest-even to binary64 / binary32 after every operation
    (the IEEE 754 definition of a correctly rounded operation), on tiny
    grids;
  * numpy scalar/array arithmetic in np.float32 / np.float64 (IEEE per-op
    rounding in the array's type; numpy never widens float32 elementwise
    ops), as the paper's Code-1 guarded per-cell sweep [Fig. 2, P:158-169]
    and as vectorised colour phases [P:198] on larger grids.
"""
from fractions import Fraction

import numpy as np
import pytest

import sor_inputs as SI


# --------------------------------------------------------------------------
# Correct rounding of an exact rational to binary64 / binary32 (round to
# nearest, ties to even), subnormals included.  Python's int/int true
# division is correctly rounded to binary64, so float(Fraction) is exact
# rounding for f64; binary32 is done by hand from the definition.
def round_f64(x: Fraction) -> Fraction:
    return Fraction(float(x))


def round_f32(x: Fraction) -> Fraction:
    if x == 0:
        return Fraction(0)
    sign = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()   # 2^e <= a < 2^(e+2)
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)                      # subnormal range: fixed quantum 2^-149
    q = Fraction(2) ** (e - 23)           # spacing of binary32 values near a
    m = a / q
    n = m.numerator // m.denominator
    rem = m - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return sign * n * q


ROUND = {"f64": round_f64, "f32": round_f32}
NPT = {"f64": np.float64, "f32": np.float32}


def exact_sor(init: np.ndarray, omega: float, iters: int, dt: str):
    """Red-black SOR on Fractions, every operation rounded to dt (readings #2-#4)."""
    rnd = ROUND[dt]
    u = [[rnd(Fraction(float(v))) for v in row] for row in init]   # step 2: u = (T)A
    w = rnd(Fraction(omega))
    q = Fraction(1, 4)
    rows, cols = len(u) - 2, len(u[0]) - 2
    last = Fraction(0)
    for _ in range(iters):
        m = Fraction(0)
        for c in (0, 1):                                        # red, then black [P:198]
            for i in range(1, rows + 1):
                for j in range(1, cols + 1):
                    if (i + j) % 2 != c:                        # colour [P:149]
                        continue
                    s = rnd(rnd(u[i - 1][j] + u[i + 1][j]) + rnd(u[i][j - 1] + u[i][j + 1]))
                    a = rnd(q * s)
                    r = rnd(a - u[i][j])
                    un = rnd(u[i][j] + rnd(w * r))
                    m = max(m, abs(rnd(un - u[i][j])))
                    u[i][j] = un
        last = m
    return np.array([[float(v) for v in row] for row in u]), float(last)


def exact_jacobi(init: np.ndarray, iters: int, dt: str):
    rnd = ROUND[dt]
    u = [[rnd(Fraction(float(v))) for v in row] for row in init]
    rows, cols = len(u) - 2, len(u[0]) - 2
    last = Fraction(0)
    for _ in range(iters):
        prev = [row[:] for row in u]                            # X_{k-1} [P:95]
        m = Fraction(0)
        for i in range(1, rows + 1):
            for j in range(1, cols + 1):
                s = rnd(rnd(prev[i - 1][j] + prev[i + 1][j]) + rnd(prev[i][j - 1] + prev[i][j + 1]))
                a = rnd(Fraction(1, 4) * s)
                m = max(m, abs(rnd(a - prev[i][j])))
                u[i][j] = a
        last = m
    return np.array([[float(v) for v in row] for row in u]), float(last)


def exact_sor3d(init: np.ndarray, omega: float, iters: int, dt: str):
    """3-D red-black SOR (reading N3-1): s = ((N+S)+(W+E))+(U+D), a = s/6
    correctly rounded, r = a - u, u' = u + w*r."""
    rnd = ROUND[dt]
    nz, ny, nx = (d - 2 for d in init.shape)
    u = {}
    for z in range(nz + 2):
        for y in range(ny + 2):
            for x in range(nx + 2):
                u[z, y, x] = rnd(Fraction(float(init[z, y, x])))
    w = rnd(Fraction(omega))
    last = Fraction(0)
    for _ in range(iters):
        m = Fraction(0)
        for c in (0, 1):
            for z in range(1, nz + 1):
                for y in range(1, ny + 1):
                    for x in range(1, nx + 1):
                        if (z + y + x) % 2 != c:
                            continue
                        ns = rnd(u[z, y - 1, x] + u[z, y + 1, x])
                        we = rnd(u[z, y, x - 1] + u[z, y, x + 1])
                        ud = rnd(u[z - 1, y, x] + u[z + 1, y, x])
                        s = rnd(rnd(ns + we) + ud)
                        a = rnd(s / 6)
                        un = rnd(u[z, y, x] + rnd(w * rnd(a - u[z, y, x])))
                        m = max(m, abs(rnd(un - u[z, y, x])))
                        u[z, y, x] = un
        last = m
    out = np.empty(init.shape)
    for k, v in u.items():
        out[k] = float(v)
    return out, float(last)


# --------------------------------------------------------------------------
# The rounding reference itself, against known binary32 facts.
def test_round_f32_definition():
    assert round_f32(Fraction(1, 3)) == Fraction(float(np.float32(1) / np.float32(3)))
    assert round_f32(Fraction(1) + Fraction(1, 2 ** 24)) == 1               # tie -> even
    assert round_f32(Fraction(1) + Fraction(3, 2 ** 24)) == 1 + Fraction(2, 2 ** 23)
    assert round_f32(Fraction(1, 2 ** 149)) == Fraction(1, 2 ** 149)        # smallest subnormal
    assert round_f32(Fraction(1, 2 ** 150)) == 0                            # tie -> even (0)
    assert round_f32(Fraction(3, 2 ** 151)) == Fraction(1, 2 ** 149)
    rng = np.random.default_rng(1)
    for _ in range(300):
        a, b = (np.float32(v) for v in rng.uniform(-50, 50, 2))
        for exact, got in ((Fraction(float(a)) + Fraction(float(b)), a + b),
                           (Fraction(float(a)) * Fraction(float(b)), a * b),
                           (Fraction(float(a)) / Fraction(float(b)), a / b)):
            assert round_f32(exact) == Fraction(float(got))


# --------------------------------------------------------------------------
# 2-D SOR: exact per-operation rounding, whole grid, both dtypes.
@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("rows,cols,omega,iters", [(3, 4, 1.37, 3), (4, 3, 1.9, 2), (2, 5, 0.376, 4)])
def test_sor_exact_rational_rounding(orc, dt, rows, cols, omega, iters):
    init = SI.random_field(rows, cols, seed=rows * 10 + cols, lo=-3.0, hi=7.0)
    exp, m = exact_sor(init, omega, iters, dt)
    u = orc.to_storage(init, dt)
    rep = orc.iterate(u, omega, iters, measure_last=True)
    assert np.array_equal(u.astype(np.float64), exp)
    assert rep.max_change == m


# Code 1: the naive guarded per-cell loop, run on numpy scalars of
# the storage type, so each operation rounds to fp32 (or fp64).
def _code1_sweep(u, w, q, iters):
    rows, cols = u.shape[0] - 2, u.shape[1] - 2
    m = u.dtype.type(0)
    for _ in range(iters):
        m = u.dtype.type(0)
        for c in (0, 1):
            for i in range(rows + 2):
                for j in range(cols + 2):
                    if i in (0, rows + 1) or j in (0, cols + 1) or (i + j) % 2 != c:
                        continue
                    s = (u[i - 1, j] + u[i + 1, j]) + (u[i, j - 1] + u[i, j + 1])
                    a = q * s
                    r = a - u[i, j]
                    un = u[i, j] + w * r
                    d = abs(un - u[i, j])
                    m = d if d > m else m
                    u[i, j] = un
    return m


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("rows,cols,omega", [(5, 7, 1.37), (8, 8, 1.93), (11, 6, 0.376), (6, 13, 1.61)])
def test_sor_code1_numpy_scalar_bitwise(orc, dt, rows, cols, omega):
    T = NPT[dt]
    init = SI.random_field(rows, cols, seed=rows * 100 + cols + 7)
    v = init.astype(T)
    m = _code1_sweep(v, T(omega), T(0.25), 4)
    u = orc.to_storage(init, dt)
    rep = orc.iterate(u, omega, 4, measure_last=True)
    assert np.array_equal(u, v)
    assert rep.max_change == float(m)


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_sor_vectorised_phases_bitwise_larger(orc, dt):
    """Colour phases as numpy array ops in the storage type (reds read only
    blacks, so a vectorised phase equals the sequential one) on a grid of a
    few thousand cells, 25 iterations, values spanning several binades."""
    T = NPT[dt]
    rows, cols, omega = 37, 45, 1.83
    init = SI.random_field(rows, cols, seed=17, lo=-40.0, hi=90.0)
    v = init.astype(T)
    i, j = np.meshgrid(np.arange(1, rows + 1), np.arange(1, cols + 1), indexing="ij")
    w, q = T(omega), T(0.25)
    for _ in range(25):
        for c in (0, 1):
            msk = ((i + j) % 2) == c
            I, J = i[msk], j[msk]
            s = (v[I - 1, J] + v[I + 1, J]) + (v[I, J - 1] + v[I, J + 1])
            v[I, J] = v[I, J] + w * (q * s - v[I, J])
    u = orc.to_storage(init, dt)
    orc.iterate(u, omega, 25)
    assert np.array_equal(u, v)


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_sor_threaded_rounding_matches_numpy(orc, dt):
    """The threaded oracle (the timed CPU baseline) rounds identically."""
    T = NPT[dt]
    init = SI.random_field(9, 11, seed=5)
    v = init.astype(T)
    _code1_sweep(v, T(1.7), T(0.25), 3)
    u = orc.to_storage(init, dt)
    orc.iterate(u, 1.7, 3, threads=3)
    assert np.array_equal(u, v)


# --------------------------------------------------------------------------
# Jacobi (NEXT-2)
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_jacobi_exact_rational_rounding(orc, dt):
    init = SI.random_field(3, 4, seed=9, lo=-2.0, hi=5.0)
    exp, m = exact_jacobi(init, 3, dt)
    u = orc.to_storage(init, dt)
    rep = orc.jacobi_iterate(u, 3, measure_last=True)
    assert np.array_equal(u.astype(np.float64), exp)
    assert rep.max_change == m


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("rows,cols", [(7, 9), (20, 13)])
def test_jacobi_numpy_bitwise(orc, dt, rows, cols):
    T = NPT[dt]
    init = SI.random_field(rows, cols, seed=rows + cols, lo=-10.0, hi=30.0)
    v = init.astype(T)
    m = T(0)
    for _ in range(12):
        p = v.copy()
        a = T(0.25) * ((p[:-2, 1:-1] + p[2:, 1:-1]) + (p[1:-1, :-2] + p[1:-1, 2:]))
        m = np.abs(a - p[1:-1, 1:-1]).max()
        v[1:-1, 1:-1] = a
    u = orc.to_storage(init, dt)
    rep = orc.jacobi_iterate(u, 12, measure_last=True)
    assert np.array_equal(u, v)
    assert rep.max_change == float(m)


# --------------------------------------------------------------------------
# 3-D (NEXT-3, reading N3-1): s/6 by correctly rounded division
def _div6_differs(s: float, dt: str) -> bool:
    rnd = ROUND[dt]
    return rnd(Fraction(s) / 6) != rnd(Fraction(s) * rnd(Fraction(1, 6)))


def test_sor3d_division_cell_where_multiply_differs(orc):
    """A single red cell whose neighbour sum s has round(s/6) != round(s*
    round(1/6)) in both dtypes; the oracle must give the division's value."""
    rng = np.random.default_rng(3)
    for dt in ("f64", "f32"):
        T = NPT[dt]
        while True:
            nb = [float(T(v)) for v in rng.uniform(0.0, 10.0, 6)]
            s = Fraction(0)
            rnd = ROUND[dt]
            s = rnd(rnd(rnd(Fraction(nb[0]) + Fraction(nb[1])) + rnd(Fraction(nb[2]) + Fraction(nb[3])))
                    + rnd(Fraction(nb[4]) + Fraction(nb[5])))
            if _div6_differs(float(s), dt):
                break
        # 1 x 1 x 2 interior: (1,1,1) black, (1,1,2) red; the red cell's six
        # neighbours are shell cells except the black (1,1,1) = nb[2]
        g = np.zeros((3, 3, 4))
        g[1, 0, 2], g[1, 2, 2] = nb[0], nb[1]              # N, S
        g[1, 1, 1], g[1, 1, 3] = nb[2], nb[3]              # W (interior black), E
        g[0, 1, 2], g[2, 1, 2] = nb[4], nb[5]              # U, D
        exp, _ = exact_sor3d(g, 1.0, 1, dt)
        u = g.astype(T)
        orc.sor3d_iterate(u, 1.0, 1)
        red = float(u[1, 1, 2])
        assert Fraction(red) == rnd(s / 6), dt              # omega = 1: u' = round(s/6)
        assert Fraction(red) != rnd(s * rnd(Fraction(1, 6))), dt
        assert np.array_equal(u.astype(np.float64), exp), dt


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_sor3d_exact_rational_rounding(orc, dt):
    init = SI.random_field3d(2, 3, 3, seed=6, lo=-1.0, hi=9.0)
    exp, m = exact_sor3d(init, 1.45, 2, dt)
    u = init.astype(NPT[dt])
    rep = orc.sor3d_iterate(u, 1.45, 2, measure_last=True)
    assert np.array_equal(u.astype(np.float64), exp)
    assert rep.max_change == m


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_sor3d_numpy_bitwise(orc, dt):
    T = NPT[dt]
    nz, ny, nx, omega = 6, 7, 9, 1.71
    init = SI.random_field3d(nz, ny, nx, seed=12, lo=-5.0, hi=50.0)
    v = init.astype(T)
    z, y, x = np.meshgrid(np.arange(1, nz + 1), np.arange(1, ny + 1), np.arange(1, nx + 1), indexing="ij")
    w, six = T(omega), T(6)
    for _ in range(10):
        for c in (0, 1):
            msk = ((z + y + x) % 2) == c
            Z, Y, X = z[msk], y[msk], x[msk]
            s = ((v[Z, Y - 1, X] + v[Z, Y + 1, X]) + (v[Z, Y, X - 1] + v[Z, Y, X + 1])) + (v[Z - 1, Y, X] + v[Z + 1, Y, X])
            u0 = v[Z, Y, X]
            v[Z, Y, X] = u0 + w * (s / six - u0)
    u = init.astype(T)
    orc.sor3d_iterate(u, omega, 10)
    assert np.array_equal(u, v)
