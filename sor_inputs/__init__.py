"""Seeded synthetic inputs for the red-black SOR hot path (shared by the oracle
tests and the GPU path).

This module holds NO arithmetic of the method (no sweep, no update, no
reduction): it only builds the initial (rows+2) x (cols+2) fp64 array (ring =
Dirichlet data, interior = initial guess) for BASELINE.json's configurations,
and the harness constant omega_opt that both sides receive by value.

Recipe (SURVEY §8(c) readings #19-#23, §8(d)):
* SplitMix64 seeded with the config's seed; U = (x >> 11) * 2**-53 in [0,1);
  value = lo + (hi - lo) * U.
* Edge traversal order: north row (i=0, j=0..cols+1), south row (i=rows+1,
  j=0..cols+1), west (j=0, i=1..rows), east (j=cols+1, i=1..rows).  Corners
  belong to the north/south rows (reading #13).
* omega_opt(N) = 2 / (1 + sin(pi / (N + 1))), computed once in fp64 (reading #18).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int) -> np.ndarray:
    """First n outputs of SplitMix64(seed) as uint64 (state += gamma; mix)."""
    k = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, n: int) -> np.ndarray:
    """U[0,1) doubles: (x >> 11) * 2**-53 (exact in fp64)."""
    return (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def omega_opt(n: int) -> float:
    """Harness constant (BASELINE.json north_star): 2 / (1 + sin(pi/(N+1)))."""
    return 2.0 / (1.0 + math.sin(math.pi / (n + 1)))


def ring_length(rows: int, cols: int) -> int:
    return 2 * (cols + 2) + 2 * rows


def set_ring(u: np.ndarray, values: np.ndarray) -> None:
    """Write ring values in the canonical traversal order N, S, W, E."""
    rows, cols = u.shape[0] - 2, u.shape[1] - 2
    w = cols + 2
    u[0, :] = values[0:w]
    u[rows + 1, :] = values[w:2 * w]
    u[1:rows + 1, 0] = values[2 * w:2 * w + rows]
    u[1:rows + 1, cols + 1] = values[2 * w + rows:2 * w + 2 * rows]


def ring_coords(rows: int, cols: int) -> tuple[np.ndarray, np.ndarray]:
    """(i, j) of every ring cell in traversal order."""
    jn = np.arange(cols + 2)
    iw = np.arange(1, rows + 1)
    i = np.concatenate([np.zeros(cols + 2, np.int64), np.full(cols + 2, rows + 1), iw, iw])
    j = np.concatenate([jn, jn, np.zeros(rows, np.int64), np.full(rows, cols + 1)])
    return i, j


def north_hot(rows: int, cols: int, north: float) -> np.ndarray:
    """C1/C3/paper: north row (corners included) = `north`, all else 0."""
    u = np.zeros((rows + 2, cols + 2), dtype=np.float64)
    u[0, :] = north
    return u


def random_edges(rows: int, cols: int, seed: int, lo: float = 0.0, hi: float = 100.0) -> np.ndarray:
    """C2/C5: every ring cell uniform [lo, hi) from SplitMix64(seed); interior 0."""
    u = np.zeros((rows + 2, cols + 2), dtype=np.float64)
    set_ring(u, lo + (hi - lo) * uniform01(seed, ring_length(rows, cols)))
    return u


def harmonic_edges(rows: int, cols: int, a: float = 0.3, b: float = 0.7, c: float = 5.0,
                   noise_seed: int | None = 4, noise: float = 1.0) -> np.ndarray:
    """C4: ring = a*x + b*y + c (+ U[0, noise) from SplitMix64(noise_seed)),
    x = j/(cols+1), y = i/(rows+1) (reading #20); interior 0."""
    u = np.zeros((rows + 2, cols + 2), dtype=np.float64)
    i, j = ring_coords(rows, cols)
    vals = a * (j / (cols + 1)) + b * (i / (rows + 1)) + c
    if noise_seed is not None and noise:
        vals = vals + noise * uniform01(noise_seed, vals.size)
    set_ring(u, vals)
    return u


def random_field(rows: int, cols: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """Every cell (ring and interior) uniform [lo, hi): for tests."""
    n = (rows + 2) * (cols + 2)
    return (lo + (hi - lo) * uniform01(seed, n)).reshape(rows + 2, cols + 2)


@dataclass(frozen=True)
class Config:
    name: str
    rows: int
    cols: int
    dtype: str                 # "f64" | "f32"
    omega: float
    kind: str                  # "north_hot" | "random_edges" | "harmonic"
    seed: int | None = None
    north: float = 100.0
    iters: int = 0             # fixed iterations (sor_iterate)
    tol: float | None = None   # then solve (sor_solve) if set
    maxit: int = 0
    check_every: int = 1
    note: str = ""
    extra: dict = field(default_factory=dict)

    def init(self) -> np.ndarray:
        if self.kind == "north_hot":
            return north_hot(self.rows, self.cols, self.north)
        if self.kind == "random_edges":
            return random_edges(self.rows, self.cols, self.seed)
        if self.kind == "harmonic":
            return harmonic_edges(self.rows, self.cols, noise_seed=self.seed)
        raise ValueError(self.kind)

    @property
    def updates_per_iter(self) -> int:
        return self.rows * self.cols


def random_shell3d(nz: int, ny: int, nx: int, seed: int, lo: float = 0.0, hi: float = 100.0) -> np.ndarray:
    """NEXT-3: (nz+2, ny+2, nx+2) fp64 array; every shell (Dirichlet) cell
    U[lo, hi) from SplitMix64(seed) in row-major order of the full array
    (interior draws discarded), interior 0."""
    u = lo + (hi - lo) * uniform01(seed, (nz + 2) * (ny + 2) * (nx + 2)).reshape(nz + 2, ny + 2, nx + 2)
    u[1:-1, 1:-1, 1:-1] = 0.0
    return np.ascontiguousarray(u)


def random_field3d(nz: int, ny: int, nx: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """NEXT-3: every cell (shell and interior) U[lo, hi) from SplitMix64(seed)."""
    return np.ascontiguousarray(
        (lo + (hi - lo) * uniform01(seed, (nz + 2) * (ny + 2) * (nx + 2))).reshape(nz + 2, ny + 2, nx + 2))


def top_hot3d(nz: int, ny: int, nx: int, top: float) -> np.ndarray:
    """NEXT-3: plane z = 0 (the whole face) = top, rest 0."""
    u = np.zeros((nz + 2, ny + 2, nx + 2))
    u[0] = top
    return u


def config(name: str, dtype: str | None = None, P: int = 1) -> Config:
    """BASELINE.json configs[0..4] as C1..C5 (+ C5W weak, PAPER = NEXT-1 replay)."""
    if name == "C1":
        return Config("C1", 64, 64, "f64", 1.5, "north_hot", north=100.0, tol=1e-6, maxit=10000,
                      note="BJ configs[0]")
    if name == "C2":
        return Config("C2", 1024, 1024, "f64", omega_opt(1024), "random_edges", seed=1, iters=2000,
                      note="BJ configs[1]")
    if name == "C3":
        return Config("C3", 4096, 4096, "f64", omega_opt(4096), "north_hot", north=100.0,
                      iters=1000, tol=1e-8, maxit=200000, note="BJ configs[2]")
    if name == "C4":
        return Config("C4", 16384, 16384, dtype or "f64", 1.9, "harmonic", seed=4, iters=500,
                      note="BJ configs[3]")
    if name == "C5":
        return Config("C5", 32768, 32768, "f64", omega_opt(32768), "random_edges", seed=7,
                      iters=200, note="BJ configs[4]")
    if name == "C5W":
        return Config("C5W", 32768 * P, 32768, "f64", omega_opt(32768), "random_edges", seed=7,
                      iters=200, note="BJ configs[4] weak scaling, 32768 rows per GPU")
    if name == "PAPER":
        return Config("PAPER", 4096, 4096, "f64", 0.376, "north_hot", north=1.0, tol=1e-5,
                      maxit=50000, check_every=4000, note="P:100, P:375, P:383 (NEXT-1)")
    raise KeyError(name)
