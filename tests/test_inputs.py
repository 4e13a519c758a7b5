"""Pins for the seeded input generator (sor_inputs), `-m "not gpu"`."""
import math

import numpy as np

import sor_inputs as SI


def test_splitmix64_reference_vector():
    # SplitMix64 (Steele, Lea, Flood 2014; Vigna's splitmix64.c) from seed 0
    z = SI.splitmix64(0, 3)
    assert [int(x) for x in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_uniform_range_and_determinism():
    a = SI.uniform01(7, 10000)
    assert a.min() >= 0.0 and a.max() < 1.0
    assert np.array_equal(a, SI.uniform01(7, 10000))
    assert not np.array_equal(a, SI.uniform01(8, 10000))
    assert abs(a.mean() - 0.5) < 0.02


def test_omega_opt_values():
    # BASELINE.json: 2/(1+sin(pi/(N+1)))
    assert SI.omega_opt(1024) == 2.0 / (1.0 + math.sin(math.pi / 1025))
    assert abs(SI.omega_opt(1024) - 1.993888803308093) < 1e-15
    assert abs(SI.omega_opt(4096) - 1.998467568850995) < 1e-15
    assert abs(SI.omega_opt(32768) - 1.999808276633988) < 1e-15


def test_ring_layout_and_traversal():
    rows, cols = 3, 4
    u = np.zeros((rows + 2, cols + 2))
    vals = np.arange(SI.ring_length(rows, cols), dtype=np.float64) + 1
    SI.set_ring(u, vals)
    assert list(u[0]) == [1, 2, 3, 4, 5, 6]           # north incl. corners
    assert list(u[-1]) == [7, 8, 9, 10, 11, 12]       # south incl. corners
    assert list(u[1:-1, 0]) == [13, 14, 15]           # west
    assert list(u[1:-1, -1]) == [16, 17, 18]          # east
    assert not u[1:-1, 1:-1].any()
    i, j = SI.ring_coords(rows, cols)
    assert np.array_equal(u[i, j], vals)


def test_configs_shapes():
    c1 = SI.config("C1")
    u = c1.init()
    assert u.shape == (66, 66) and (u[0] == 100).all() and u[1:].sum() == 0
    c2 = SI.config("C2")
    u = c2.init()
    assert u.shape == (1026, 1026)
    assert 0 <= u.min() and u.max() < 100 and not u[1:-1, 1:-1].any()
    c4 = SI.config("C4")
    assert c4.omega == 1.9 and c4.iters == 500
    h = SI.harmonic_edges(30, 40)
    assert 5.0 <= h[0].min() and h[-1].max() < 7.0
    assert SI.config("C5W", P=2).rows == 65536
