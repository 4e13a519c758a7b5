"""Pins for the CPU oracle, all `-m "not gpu"`.

Each test pins the oracle to something other than itself: hand-evaluated
values (tests/golden/), closed forms of classical SOR theory, invariants,
special cases that reduce to a textbook routine written independently here,
brute force (dense direct solve, naive per-cell loops).  A plausible mistake
anywhere in oracle/sor_oracle.c (dropped term, wrong sign, wrong colour
origin, transposed operand, wrong phase order, wrong cadence) fails at least
one of them.
"""
import math
import os

import numpy as np
import pytest

import sor_inputs as SI

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------
# P1: hand-computed first iteration of C1 (bitwise; dyadic values)
def _golden_c1():
    rows = []
    with open(os.path.join(GOLDEN, "c1_iteration1.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            ph, i, j, v = line.split()
            rows.append((ph, int(i), int(j), float(v)))
    return rows


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_p1_c1_first_iteration_hand_values(orc, dtype):
    cfg = SI.config("C1")
    u = orc.to_storage(cfg.init(), dtype)
    gold = _golden_c1()
    if dtype == "f64":
        # red phase alone (orc_half_sweep), then black
        m = orc.half_sweep(u, 0, cfg.omega)
        for ph, i, j, v in gold:
            if ph == "red":
                assert u[i, j] == v, (i, j)
        m = max(m, orc.half_sweep(u, 1, cfg.omega))
        for ph, i, j, v in gold:
            if ph == "black":
                assert u[i, j] == v, (i, j)
            if ph == "maxdelta":
                assert m == v
    u2 = orc.to_storage(cfg.init(), dtype)
    rep = orc.iterate(u2, cfg.omega, 1, measure_last=True)
    assert rep.iters == 1 and rep.half_sweeps == 2
    for ph, i, j, v in gold:
        if ph == "black":
            assert u2[i, j] == v, (dtype, i, j)
        if ph == "maxdelta":
            assert rep.max_change == v
    # ring untouched
    assert np.array_equal(u2[0], cfg.init()[0].astype(u2.dtype))
    assert not u2[-1].any() and not u2[1:, 0].any() and not u2[1:, -1].any()


# --------------------------------------------------------------------------
# P2: SPEC worked examples
def test_p2_cell_update_examples(orc):
    # X=0, neighbours (1,0,0,0), omega=0.376 -> 0.094
    assert orc.cell_update(1.0, 0.0, 0.0, 0.0, 0.0, 0.376) == 0.094
    # omega=1, X=0.5, neighbours (1,1,1,1) -> 1.0 (pure GS iterate)
    assert orc.cell_update(1.0, 1.0, 1.0, 1.0, 0.5, 1.0) == 1.0
    # zero neighbourhood is a fixed point for any omega
    for w in (0.376, 1.0, 1.9):
        assert orc.cell_update(0.0, 0.0, 0.0, 0.0, 0.0, w) == 0.0
    # Eq. 1 form omega*Xbar + (1-omega)*X agrees with the BJ form up to rounding
    rng = np.random.default_rng(5)
    for _ in range(200):
        n, s, w_, e, u = rng.uniform(-10, 10, 5)
        om = rng.uniform(0.05, 1.95)
        eq1 = om * ((n + s + w_ + e) / 4.0) + (1.0 - om) * u
        assert abs(orc.cell_update(n, s, w_, e, u, om) - eq1) <= 1e-13 * 40


def test_p2_red_sweep_n4(orc):
    # n=4 (2x2 interior), north=1, red sweep omega=0.376:
    # interior red cells adjacent to north become 0.094, black cells stay 0.
    u = SI.north_hot(2, 2, 1.0)
    orc.half_sweep(u, 0, 0.376)
    assert u[1, 1] == 0.094          # (1,1) red, touches north
    assert u[2, 2] == 0.0            # (2,2) red, not adjacent to north
    assert u[1, 2] == 0.0 and u[2, 1] == 0.0   # black untouched


def test_p2_jacobi_one_step_n4(orc):
    # one Jacobi step on n=4 north-hot grid -> cells next to north 0.25
    u = SI.north_hot(2, 2, 1.0)
    rep = orc.jacobi(u, 1e-300, 1)
    assert rep.iters == 1
    assert u[1, 1] == 0.25 and u[1, 2] == 0.25
    assert u[2, 1] == 0.0 and u[2, 2] == 0.0


# --------------------------------------------------------------------------
# Brute force: naive Code-1 style guarded per-cell sweep
def _naive_iteration(u, omega):
    rows, cols = u.shape[0] - 2, u.shape[1] - 2
    for c in (0, 1):
        for i in range(rows + 2):
            for j in range(cols + 2):
                if i in (0, rows + 1) or j in (0, cols + 1):
                    continue
                if (i + j) % 2 == c:          # Code 1: `if ((i+j) % 2 == c)` (reading #14)
                    s = (u[i - 1, j] + u[i + 1, j]) + (u[i, j - 1] + u[i, j + 1])
                    u[i, j] = u[i, j] + omega * (0.25 * s - u[i, j])


@pytest.mark.parametrize("rows,cols", [(1, 1), (1, 5), (4, 1), (5, 7), (6, 6), (9, 4)])
def test_stride2_equals_naive_guarded(orc, rows, cols):
    u = SI.random_field(rows, cols, seed=rows * 100 + cols)
    v = u.copy()
    for _ in range(3):
        _naive_iteration(v, 1.37)
    orc.iterate(u, 1.37, 3)
    assert np.array_equal(u, v)


# --------------------------------------------------------------------------
# P3: fixed point = dense direct solve of the 5-point Dirichlet system
@pytest.mark.parametrize("rows,cols", [(7, 7), (5, 9), (12, 3), (16, 16)])
def test_p3_converges_to_dense_solution(orc, rows, cols):
    init = SI.random_edges(rows, cols, seed=rows + 31 * cols)
    bnd = np.abs(init).max()
    exact = init.copy()
    orc.dense_solve(exact)
    u = init.copy()
    w = SI.omega_opt(max(rows, cols))
    rep = orc.solve(u, w, 1e-15 * bnd, 100000)
    assert rep.converged
    assert np.abs(u - exact).max() <= 1e-12 * bnd


def test_p3_jacobi_and_sor_agree(orc):
    # converged Jacobi vs converged SOR within 10*eps
    init = SI.north_hot(15, 15, 1.0)
    a = init.copy()
    b = init.copy()
    ra = orc.jacobi(a, 1e-12, 200000)
    rb = orc.solve(b, 1.0, 1e-12, 200000)
    assert ra.converged and rb.converged
    exact = init.copy()
    orc.dense_solve(exact)
    assert np.abs(a - b).max() <= 1e-9
    assert np.abs(a - exact).max() <= 1e-9


# --------------------------------------------------------------------------
# P4: discrete-harmonic boundary is a fixed point
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("omega", [0.376, 1.0, 1.5, 1.9])
def test_p4_dyadic_linear_fixed_point_bitwise(orc, dtype, omega):
    rows, cols = 13, 10
    i, j = np.meshgrid(np.arange(rows + 2), np.arange(cols + 2), indexing="ij")
    lin = 0.25 * j + 0.75 * i + 5.0
    u = orc.to_storage(lin, dtype)
    ref = u.copy()
    orc.iterate(u, omega, 200)
    assert np.array_equal(u, ref)


def test_p4_c4_base_drift_and_convergence(orc):
    rows = cols = 24
    u = SI.harmonic_edges(rows, cols, noise_seed=None)   # 0.3x + 0.7y + 5, no noise
    i, j = np.meshgrid(np.arange(rows + 2), np.arange(cols + 2), indexing="ij")
    exact = 0.3 * (j / (cols + 1)) + 0.7 * (i / (rows + 1)) + 5.0
    # starting AT the linear function: it is (to rounding) a fixed point
    v = exact.copy()
    orc.iterate(v, 1.9, 500)
    assert np.abs(v - exact).max() <= 1e-13
    # from interior 0: converges to the linear function
    rep = orc.solve(u, SI.omega_opt(rows), 1e-14, 100000)
    assert rep.converged
    assert np.abs(u - exact).max() <= 1e-12


# --------------------------------------------------------------------------
# P5: omega = 1 is red-black Gauss-Seidel (independent textbook GS in numpy)
def _textbook_rb_gs(u, iters):
    rows, cols = u.shape[0] - 2, u.shape[1] - 2
    i, j = np.meshgrid(np.arange(1, rows + 1), np.arange(1, cols + 1), indexing="ij")
    for _ in range(iters):
        for c in (0, 1):
            m = ((i + j) % 2) == c
            I, J = i[m], j[m]
            u[I, J] = 0.25 * ((u[I - 1, J] + u[I + 1, J]) + (u[I, J - 1] + u[I, J + 1]))


@pytest.mark.parametrize("n", [17, 18])
def test_p5_omega1_is_gauss_seidel(orc, n):
    init = SI.random_edges(n, n, seed=n)
    bnd = np.abs(init).max()
    a, b = init.copy(), init.copy()
    for k in range(40):
        orc.iterate(a, 1.0, 1)
        _textbook_rb_gs(b, 1)
        assert np.abs(a - b).max() <= 1e-13 * bnd, k


# --------------------------------------------------------------------------
# P6: asymptotic convergence factor vs Young's closed form
def _young_rho(omega, n):
    mu = math.cos(math.pi / (n + 1))
    wopt = 2.0 / (1.0 + math.sqrt(1.0 - mu * mu))
    if omega >= wopt:
        return omega - 1.0
    return ((omega * mu + math.sqrt(omega * omega * mu * mu - 4.0 * (omega - 1.0))) / 2.0) ** 2


def _delta_history(orc, n, omega, iters, seed=3):
    u = np.zeros((n + 2, n + 2))
    u[1:-1, 1:-1] = SI.uniform01(seed, n * n).reshape(n, n)
    hist = []
    for _ in range(iters):
        hist.append(orc.iterate(u, omega, 1, measure_last=True).max_change)
    return np.array(hist)


@pytest.mark.parametrize("n,omega", [(32, 1.0), (32, 1.5), (16, 1.2)])
def test_p6_rho_below_omega_opt(orc, n, omega):
    h = _delta_history(orc, n, omega, 2500)
    ratio = h[-1] / h[-2]
    assert ratio == pytest.approx(_young_rho(omega, n), rel=2e-5)


@pytest.mark.parametrize("n,omega", [(16, None), (32, 1.95), (64, None)])
def test_p6_rho_at_or_above_omega_opt(orc, n, omega):
    w = SI.omega_opt(n) if omega is None else omega
    h = _delta_history(orc, n, w, 700)
    # complex eigenvalues: the ratio oscillates; use the geometric mean over a window
    lo, hi = 300, 650
    gm = (h[hi] / h[lo]) ** (1.0 / (hi - lo))
    assert h[hi] > 1e-250
    assert gm == pytest.approx(w - 1.0, rel=5e-3)


# --------------------------------------------------------------------------
# P7: symmetry
def test_p7_mirror_symmetry_odd_cols(orc):
    rows, cols = 20, 33
    u = np.zeros((rows + 2, cols + 2))
    e = SI.uniform01(11, cols + 2) * 100
    u[0, :] = (e + e[::-1]) / 2          # left-right symmetric north edge
    u[1:-1, 0] = u[1:-1, -1] = 7.0
    orc.iterate(u, 1.7, 60)
    assert np.array_equal(u, u[:, ::-1])


def test_p7_centre_value_odd_n(orc):
    # four rotated north-hot problems superpose to the all-T solution: centre = T/4
    n = 33
    u = SI.north_hot(n, n, 100.0)
    u[0, 0] = u[0, -1] = 0.0             # corners are never read
    rep = orc.solve(u, SI.omega_opt(n), 1e-12, 100000)
    assert rep.converged
    assert abs(u[17, 17] - 25.0) <= 1e-9


def test_p7_even_n_central_cells_sum(orc):
    n = 32
    u = SI.north_hot(n, n, 100.0)
    rep = orc.solve(u, SI.omega_opt(n), 1e-12, 100000)
    assert rep.converged
    assert abs(u[16, 16] + u[16, 17] + u[17, 16] + u[17, 17] - 100.0) <= 1e-8


# --------------------------------------------------------------------------
# P8: maximum principle for 0 < omega <= 1
@pytest.mark.parametrize("omega", [0.376, 0.8, 1.0])
def test_p8_maximum_principle(orc, omega):
    u = SI.random_field(23, 17, seed=99)
    for _ in range(30):
        orc.iterate(u, omega, 1)
        assert u.min() >= 0.0 and u.max() <= 1.0


# --------------------------------------------------------------------------
# P10: the paper's own protocol (NEXT-1) obeys the diffusion similarity law.
# North edge 1, interior 0, omega = 0.376 [P:100], checks every K = 4000
# iterations, eps = 1e-5 [P:383].  Under-relaxed SOR from a step boundary is
# a discrete heat equation; its continuum limit is u = erfc(y / 2 sqrt(D k)),
# whose largest per-iteration change is max_y du/dk = 1 / (sqrt(2 pi e) k)
# whatever the diffusivity D.  So the checked max-changes must follow
# 0.24197 / k and the stop test (strict <) first passes at k = 28000 (the
# first multiple of 4000 above 1/(sqrt(2 pi e) 1e-5) = 24197).  512 x 512 is
# deep enough that the front (~3 sqrt(D k) ~ 220 rows at k = 28000) stays
# away from the far ring.
def test_p10_paper_protocol_similarity_law(orc):
    c = 1.0 / math.sqrt(2.0 * math.pi * math.e)
    threads = max(1, min(16, len(os.sched_getaffinity(0))))
    u = SI.north_hot(512, 512, 1.0)
    for m in range(1, 8):
        k = 4000 * m
        rep = orc.iterate(u, 0.376, 4000, measure_last=True, threads=threads)
        assert abs(rep.max_change * k / c - 1.0) < 5e-3, (k, rep.max_change)
    u = SI.north_hot(512, 512, 1.0)
    rep = orc.solve(u, 0.376, 1e-5, 50000, check_every=4000, threads=threads)
    assert rep.converged and rep.iters == 28000 and rep.checks == 7
    assert rep.max_change < 1e-5 and abs(rep.max_change * 28000 / c - 1.0) < 5e-3


# --------------------------------------------------------------------------
# P9 / P15: cadence and accounting
def test_p9_zero_problem_converges_at_first_check(orc):
    u = np.zeros((10, 12))
    rep = orc.solve(u, 1.5, 1e-6, 100, check_every=7)
    assert rep.converged and rep.iters == 7 and rep.max_change == 0.0 and rep.checks == 1


def test_p15_check_accounting(orc):
    u = SI.north_hot(8, 8, 1.0)
    rep = orc.solve(u, 0.376, 1e-300, 20, check_every=7)
    assert not rep.converged
    assert rep.iters == 20 and rep.half_sweeps == 40 and rep.checks == 2   # checks at 7 and 14


def test_solve_strict_less_than(orc):
    # equality continues (reading #7): tol equal to the exact max change must not stop
    cfg = SI.config("C1")
    u = cfg.init()
    rep = orc.solve(u, cfg.omega, 65.625, 5)       # iteration-1 change is exactly 65.625
    assert rep.iters >= 2
    u = cfg.init()
    rep = orc.solve(u, cfg.omega, np.nextafter(65.625, 1e9), 5)
    assert rep.converged and rep.iters == 1


def test_oracle_rejects_bad_args(orc):
    u = np.zeros((5, 5))
    with pytest.raises(ValueError):
        orc.solve(u, 2.0, 1e-6, 10)
    with pytest.raises(ValueError):
        orc.solve(u, 1.0, 0.0, 10)
    with pytest.raises(ValueError):
        orc.solve(u, 1.0, 1e-6, 10, check_every=11)


# --------------------------------------------------------------------------
# P13: fused |delta| == Algorithm 1's snapshot diff, bitwise
@pytest.mark.parametrize("K", [1, 3, 50])
def test_p13_fused_delta_equals_snapshot(orc, K):
    init = SI.random_edges(21, 18, seed=K)
    a, b = init.copy(), init.copy()
    ra = orc.solve(a, 1.8, 1e-4, 400, check_every=K)
    rb = orc.solve_snapshot(b, 1.8, 1e-4, 400, check_every=K)
    assert (ra.status, ra.iters, ra.checks) == (rb.status, rb.iters, rb.checks)
    assert ra.max_change == rb.max_change
    assert np.array_equal(a, b)


# --------------------------------------------------------------------------
# P14: threaded (P workers + barrier per phase) == serial, bitwise
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("P", [2, 3, 8])
def test_p14_threads_equal_serial(orc, dtype, P):
    init = SI.random_edges(37, 29, seed=P)
    a, b = orc.to_storage(init, dtype), orc.to_storage(init, dtype)
    ra = orc.solve(a, 1.9, 1e-3, 300)
    rb = orc.solve(b, 1.9, 1e-3, 300, threads=P)
    assert (ra.status, ra.iters, ra.max_change) == (rb.status, rb.iters, rb.max_change)
    assert np.array_equal(a, b)
    ia, ib = orc.to_storage(init, dtype), orc.to_storage(init, dtype)
    orc.iterate(ia, 1.3, 17)
    orc.iterate(ib, 1.3, 17, threads=P)
    assert np.array_equal(ia, ib)


def test_partition_rows(orc):
    for rows in (1, 7, 64, 100):
        for P in (1, 2, 3, 8):
            if P > rows:
                continue
            spans = [orc.partition_rows(rows, P, p) for p in range(P)]
            assert spans[0][0] == 1 and spans[-1][1] == rows + 1
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
            assert all(spans[p][1] == spans[p + 1][0] for p in range(P - 1))


# --------------------------------------------------------------------------
# slab emulation: a slab with halo rows as its ring, row_off = global offset
def test_row_offset_slab_equivalence(orc):
    rows, cols = 20, 11
    g = SI.random_field(rows, cols, seed=4)
    ref = g.copy()
    orc.half_sweep(ref, 0, 1.6)
    # rows 6..13 (global) as a slab whose ring rows are global rows 5 and 14
    s = g[5:15].copy()
    orc.half_sweep(s, 0, 1.6, row_off=5)
    assert np.array_equal(s[1:-1], ref[6:14])


# --------------------------------------------------------------------------
# fp32: subnormals preserved (reading #17), f32 tracks f64
def test_f32_subnormals_kept(orc):
    u = np.zeros((12, 12), dtype=np.float32)
    u[0, :] = np.float32(2e-38)
    orc.iterate(u, 1.0, 5)
    tiny = u[(u != 0) & (np.abs(u) < np.finfo(np.float32).tiny)]
    assert tiny.size > 0


def test_f32_tracks_f64(orc):
    init = SI.random_edges(30, 30, seed=8)
    a, b = orc.to_storage(init, "f64"), orc.to_storage(init, "f32")
    orc.iterate(a, 1.9, 100)
    orc.iterate(b, 1.9, 100)
    assert np.abs(a - b.astype(np.float64)).max() <= 1e-4 * 100


def test_nan_propagates_in_max(orc):
    u = SI.north_hot(6, 6, 1.0)
    u[0, 3] = np.nan
    rep = orc.iterate(u, 1.0, 1, measure_last=True)
    assert math.isnan(rep.max_change)
    u = SI.north_hot(6, 6, 1.0)
    u[0, 3] = np.nan
    rep = orc.solve(u, 1.0, 1e-3, 5)
    assert not rep.converged


# --------------------------------------------------------------------------
# NEXT-2: Jacobi in both modes
def test_jacobi_one_step_s187(orc):
    """from a north-hot n=4 grid (interior 0), one Jacobi step gives
    0.25 * north in the row next to the north edge and 0 elsewhere."""
    for dtype in (np.float64, np.float32):
        u = SI.north_hot(4, 4, 1.0).astype(dtype)
        rep = orc.jacobi_iterate(u, 1, measure_last=True)
        assert np.array_equal(u[1, 1:-1], np.full(4, 0.25, dtype))
        assert not u[2:-1, 1:-1].any() and rep.max_change == 0.25 and rep.half_sweeps == 1


def test_jacobi_reads_only_the_previous_iterate(orc):
    """Out-of-place semantics: the second step uses only step-1 values.  Row 1
    after two steps: 0.25*(1 + 0.25) at the ends, 0.25*(1 + 0.25 + 0.25*... ) --
    written out from the neighbours of step 1 (not a re-typed loop: the
    step-1 field is the closed form 0.25 on row 1)."""
    u = SI.north_hot(4, 4, 1.0)
    orc.jacobi_iterate(u, 2)
    # step 1: row 1 = 0.25, rest 0.  step 2: row 1 = 0.25*(1 + 0 + W + E), row 2 = 0.25*0.25
    assert u[1, 1] == 0.25 * (1.0 + 0.25) and u[1, 2] == 0.25 * (1.0 + 0.5)
    assert np.array_equal(u[2, 1:-1], np.full(4, 0.0625)) and not u[3:-1, 1:-1].any()


def test_jacobi_fixed_point_is_dense_solution(orc):
    u = SI.random_edges(9, 7, seed=3)
    ref = u.copy()
    orc.dense_solve(ref)
    rep = orc.jacobi_solve(u, 1e-15 * 100, 200000, 1)
    assert rep.converged
    assert np.abs(u - ref).max() <= 1e-10 * 100


def test_jacobi_dyadic_linear_field_bitwise_fixed_point(orc):
    rows, cols = 13, 10
    i, j = np.meshgrid(np.arange(rows + 2), np.arange(cols + 2), indexing="ij")
    u = 0.25 * j + 0.75 * i + 5.0
    for dtype in (np.float64, np.float32):
        v = u.astype(dtype)
        w = v.copy()
        orc.jacobi_iterate(w, 50)
        assert np.array_equal(w, v)


@pytest.mark.parametrize("n", [16, 24])
def test_jacobi_asymptotic_rate_is_cos_pi_over_n_plus_1(orc, n):
    """Jacobi's iteration matrix has spectral radius mu = cos(pi/(N+1)) with
    eigenvalues +mu and -mu both present: the checked max-changes decay at
    |mu| per iteration (geometric mean over a window)."""
    mu = math.cos(math.pi / (n + 1))
    u = np.zeros((n + 2, n + 2))
    u[1:-1, 1:-1] = SI.random_field(n, n, seed=5)[1:-1, 1:-1]
    hist = [orc.jacobi_iterate(u, 1, measure_last=True).max_change for _ in range(1500)]
    a, b = 1000, 1400
    rate = (hist[b] / hist[a]) ** (1.0 / (b - a))
    assert abs(rate - mu) < 2e-4, (rate, mu)


def test_jacobi_cadence_and_modes_agree(orc):
    """Checks at multiples of K only; solve with K=1 equals the
    original Jacobi routine used by the P3 pin, bitwise."""
    u = SI.random_edges(20, 17, seed=8)
    v = u.copy()
    rep = orc.jacobi_solve(u, 1e-3, 5000, 1)
    rep2 = orc.jacobi(v, 1e-3, 5000)
    assert (rep.iters, rep.max_change) == (rep2.iters, rep2.max_change) and np.array_equal(u, v)
    w = SI.random_edges(20, 17, seed=8)
    rep3 = orc.jacobi_solve(w, 1e-3, 5000, 7)
    assert rep3.iters % 7 == 0 and rep3.iters >= rep.iters and rep3.checks == rep3.iters // 7
    z = SI.north_hot(8, 8, 1.0)
    rep4 = orc.jacobi_solve(z, 1e-300, 20, 7)
    assert not rep4.converged and rep4.iters == 20 and rep4.checks == 2


# --------------------------------------------------------------------------
# NEXT-3: 3-D red-black SOR (7-point, P:410 future work)
def test_sor3d_fixed_point_is_dense_7point_solution(orc):
    u = SI.random_shell3d(5, 6, 7, seed=4)
    ref = u.copy()
    orc.dense_solve3d(ref)
    rep = orc.sor3d_solve(u, 1.5, 1e-14 * 100, 100000, 1)
    assert rep.converged
    assert np.abs(u - ref).max() <= 1e-11 * 100


@pytest.mark.parametrize("omega", [1.0, 1.5])
def test_sor3d_rate_matches_young(orc, omega):
    """Red-black ordering of the 7-point Laplacian is consistently ordered: the
    3-D Jacobi radius on an N^3 cube is mu = cos(pi/(N+1)) and Young's formula
    gives SOR's rate below omega_opt (P6 in 3-D)."""
    n = 12
    mu = math.cos(math.pi / (n + 1))
    rho = ((omega * mu + math.sqrt(omega * omega * mu * mu - 4 * (omega - 1))) / 2) ** 2
    u = SI.random_field3d(n, n, n, seed=3)
    u[0], u[-1], u[:, 0], u[:, -1], u[:, :, 0], u[:, :, -1] = 0, 0, 0, 0, 0, 0
    hist = [orc.sor3d_iterate(u, omega, 1, measure_last=True).max_change for _ in range(400)]
    a, b = 300, 390
    rate = (hist[b] / hist[a]) ** (1.0 / (b - a))
    assert abs(rate - rho) < 2e-3 * rho, (rate, rho)


def test_sor3d_red_first_hand_values(orc):
    """Top face 1, interior 0, one iteration: red (z+y+x even) first.  Red
    (1,1,2) sees only the top: omega/6.  Black (1,1,1) then sees the top and
    the two new red neighbours (1,1,2), (1,2,1): omega*(1 + 2 omega/6)/6.
    Exact rational values, compared within a few ulps; with the colours
    swapped both values change at first order."""
    from fractions import Fraction as F
    w = 1.5
    u = SI.top_hot3d(4, 4, 4, 1.0)
    orc.sor3d_iterate(u, w, 1)
    red = F(3, 2) / 6
    black = F(3, 2) * (1 + 2 * red) / 6
    assert abs(u[1, 1, 2] - float(red)) <= 4e-16 and abs(u[1, 1, 1] - float(black)) <= 4e-16
    assert u[2, 1, 1] == 0.0 and u[3, 1, 2] == 0.0


def test_sor3d_mirror_symmetry_and_f32(orc):
    u = SI.random_shell3d(6, 5, 9, seed=8)
    u[:, :, ::-1] = u  # symmetric under x -> nx+1-x (nx odd keeps colours)
    u = np.ascontiguousarray((u + u[:, :, ::-1]) / 2)
    orc.sor3d_iterate(u, 1.8, 25)
    assert np.array_equal(u, u[:, :, ::-1])
    v = SI.random_shell3d(6, 5, 9, seed=8)
    w = v.astype(np.float32)
    orc.sor3d_iterate(v, 1.8, 25)
    orc.sor3d_iterate(w, 1.8, 25)
    assert np.abs(w - v).max() <= 1e-5 * 100
