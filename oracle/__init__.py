"""CPU oracle for red-black SOR (arXiv 1401.0763) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1401_0763_b200``) never imports it and shares no code with it.

The arithmetic lives in ``sor_oracle.c`` (plain C11, -ffp-contract=off); this
module only compiles it and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sor_oracle.c")
HDR = os.path.join(HERE, "sor_oracle.h")
LIB = os.path.join(HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
          "-Wall", "-Wextra", "-Wno-unused-parameter"]


def build_oracle(force: bool = False) -> str:
    """Compile liboracle.so in-tree (gcc; no FMA contraction, no fast-math)."""
    stale = (not os.path.exists(LIB)
             or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(HDR)))
    if force or stale:
        tmp = LIB + ".tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm", "-lpthread"])
        os.replace(tmp, LIB)
    return LIB


class _Report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iters", ctypes.c_int64),
                ("max_change", ctypes.c_double), ("half_sweeps", ctypes.c_int64),
                ("checks", ctypes.c_int64)]


@dataclass
class Report:
    status: int          # 0 done/converged, 1 not converged
    iters: int
    max_change: float
    half_sweeps: int
    checks: int

    @property
    def converged(self) -> bool:
        return self.status == 0


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_oracle())
        i64, dbl, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_int
        vp = ctypes.c_void_p
        rp = ctypes.POINTER(_Report)
        _lib.orc_cell_update_f64.restype = dbl
        _lib.orc_cell_update_f64.argtypes = [dbl] * 6
        _lib.orc_cell_update_f32.restype = ctypes.c_float
        _lib.orc_cell_update_f32.argtypes = [ctypes.c_float] * 5 + [dbl]
        for name in ("orc_sor_run_f64", "orc_sor_run_f32"):
            f = getattr(_lib, name)
            f.restype = i32
            f.argtypes = [vp, i64, i64, i64, dbl, i32, i64, dbl, i64, i32, rp]
        for name in ("orc_sor_run_threads_f64", "orc_sor_run_threads_f32"):
            f = getattr(_lib, name)
            f.restype = i32
            f.argtypes = [vp, i64, i64, dbl, i32, i64, dbl, i64, i32, i32, rp]
        _lib.orc_half_sweep_f64.restype = None
        _lib.orc_half_sweep_f64.argtypes = [vp, i64, i64, i64, i32, dbl, ctypes.POINTER(dbl)]
        _lib.orc_sor_run_snapshot_f64.restype = i32
        _lib.orc_sor_run_snapshot_f64.argtypes = [vp, i64, i64, dbl, i64, dbl, i64, rp]
        _lib.orc_partition_rows.restype = None
        _lib.orc_partition_rows.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        for name in ("orc_jacobi_run_f64", "orc_jacobi_run_f32"):
            f = getattr(_lib, name)
            f.restype = i32
            f.argtypes = [vp, i64, i64, i32, i64, dbl, i64, i32, rp]
        for name in ("orc_sor3d_run_f64", "orc_sor3d_run_f32"):
            f = getattr(_lib, name)
            f.restype = i32
            f.argtypes = [vp, i64, i64, i64, dbl, i32, i64, dbl, i64, i32, rp]
        _lib.orc_dense_solve3d_f64.restype = i32
        for name in ("orc_variant_run_f64", "orc_variant_run_f32"):
            f = getattr(_lib, name)
            f.restype = i32
            f.argtypes = [vp, i64, i64, i32, i64, i64, i64, dbl, i32, i64, dbl, i64, i32, rp]
        _lib.orc_dense_solve3d_f64.argtypes = [vp, i64, i64, i64]
        _lib.orc_jacobi_f64.restype = i32
        _lib.orc_jacobi_f64.argtypes = [vp, i64, i64, i64, dbl, rp]
        _lib.orc_dense_solve_f64.restype = i32
        _lib.orc_dense_solve_f64.argtypes = [vp, i64, i64]
    return _lib


def _grid(u: np.ndarray, dtype) -> np.ndarray:
    assert u.ndim == 2 and u.dtype == dtype and u.flags.c_contiguous
    return u


def _rep(r: _Report) -> Report:
    return Report(int(r.status), int(r.iters), float(r.max_change), int(r.half_sweeps), int(r.checks))


def to_storage(init: np.ndarray, dtype: str) -> np.ndarray:
    """Step 2 of the oracle algorithm: u = (T)A (round-to-nearest for f32)."""
    if dtype == "f64":
        return np.array(init, dtype=np.float64, copy=True, order="C")
    if dtype == "f32":
        return np.array(init, dtype=np.float32, copy=True, order="C")
    raise ValueError(dtype)


def iterate(u: np.ndarray, omega: float, iters: int, measure_last: bool = False,
            row_off: int = 0, threads: int = 1) -> Report:
    """Run exactly `iters` red-black iterations in place (Algorithm 1 without the stop test)."""
    return _run(u, omega, 0, iters, 1.0, 1, measure_last, row_off, threads)


def solve(u: np.ndarray, omega: float, tol: float, maxit: int, check_every: int = 1,
          threads: int = 1) -> Report:
    """Algorithm 1: iterate until a checked max|delta| < tol or maxit."""
    return _run(u, omega, 1, maxit, tol, check_every, False, 0, threads)


def _run(u, omega, mode, n_iter, tol, K, measure_last, row_off, threads) -> Report:
    rows, cols = u.shape[0] - 2, u.shape[1] - 2
    r = _Report()
    L = lib()
    if u.dtype == np.float64:
        if threads == 1:
            L.orc_sor_run_f64(u.ctypes.data, rows, cols, row_off, omega, mode, n_iter, tol, K,
                              int(measure_last), ctypes.byref(r))
        else:
            assert row_off == 0
            L.orc_sor_run_threads_f64(u.ctypes.data, rows, cols, omega, mode, n_iter, tol, K,
                                      int(measure_last), threads, ctypes.byref(r))
    elif u.dtype == np.float32:
        if threads == 1:
            L.orc_sor_run_f32(u.ctypes.data, rows, cols, row_off, omega, mode, n_iter, tol, K,
                              int(measure_last), ctypes.byref(r))
        else:
            assert row_off == 0
            L.orc_sor_run_threads_f32(u.ctypes.data, rows, cols, omega, mode, n_iter, tol, K,
                                      int(measure_last), threads, ctypes.byref(r))
    else:
        raise TypeError(u.dtype)
    if r.status < 0:
        raise ValueError("oracle rejected arguments")
    return _rep(r)


def half_sweep(u: np.ndarray, colour: int, omega: float, row_off: int = 0) -> float:
    _grid(u, np.float64)
    m = ctypes.c_double(0.0)
    lib().orc_half_sweep_f64(u.ctypes.data, u.shape[0] - 2, u.shape[1] - 2, row_off, colour,
                             omega, ctypes.byref(m))
    return m.value


def solve_snapshot(u: np.ndarray, omega: float, tol: float, maxit: int, check_every: int) -> Report:
    _grid(u, np.float64)
    r = _Report()
    lib().orc_sor_run_snapshot_f64(u.ctypes.data, u.shape[0] - 2, u.shape[1] - 2, omega, maxit,
                                   tol, check_every, ctypes.byref(r))
    return _rep(r)


def partition_rows(rows: int, P: int, p: int) -> tuple[int, int]:
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    lib().orc_partition_rows(rows, P, p, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def jacobi(u: np.ndarray, tol: float, maxit: int) -> Report:
    _grid(u, np.float64)
    r = _Report()
    lib().orc_jacobi_f64(u.ctypes.data, u.shape[0] - 2, u.shape[1] - 2, maxit, tol, ctypes.byref(r))
    return _rep(r)


def _jacobi_run(u, mode, n_iter, tol, K, measure_last) -> Report:
    f64 = u.dtype == np.float64
    _grid(u, np.float64 if f64 else np.float32)
    r = _Report()
    fn = lib().orc_jacobi_run_f64 if f64 else lib().orc_jacobi_run_f32
    fn(u.ctypes.data, u.shape[0] - 2, u.shape[1] - 2, mode, n_iter, tol, K, int(measure_last), ctypes.byref(r))
    return _rep(r)


def jacobi_iterate(u: np.ndarray, iters: int, measure_last: bool = False) -> Report:
    """NEXT-2: exactly `iters` Jacobi iterations in place (float64 or float32 storage)."""
    return _jacobi_run(u, 0, iters, 1.0, 1, measure_last)


def jacobi_solve(u: np.ndarray, tol: float, maxit: int, check_every: int = 1) -> Report:
    """NEXT-2: Jacobi with Algorithm 1's loop control (check every K, strict <)."""
    return _jacobi_run(u, 1, maxit, tol, check_every, False)


def _sor3d(u, omega, mode, n_iter, tol, K, measure_last) -> Report:
    f64 = u.dtype == np.float64
    assert u.ndim == 3 and u.flags.c_contiguous and u.dtype in (np.float64, np.float32)
    r = _Report()
    fn = lib().orc_sor3d_run_f64 if f64 else lib().orc_sor3d_run_f32
    fn(u.ctypes.data, u.shape[0] - 2, u.shape[1] - 2, u.shape[2] - 2, omega, mode, n_iter, tol, K,
       int(measure_last), ctypes.byref(r))
    return _rep(r)


def sor3d_iterate(u: np.ndarray, omega: float, iters: int, measure_last: bool = False) -> Report:
    """NEXT-3: 3-D red-black SOR, `iters` iterations in place ((nz+2, ny+2, nx+2) array)."""
    return _sor3d(u, omega, 0, iters, 1.0, 1, measure_last)


def sor3d_solve(u: np.ndarray, omega: float, tol: float, maxit: int, check_every: int = 1) -> Report:
    return _sor3d(u, omega, 1, maxit, tol, check_every, False)


def _variant(u, kind, p1, p2, p3, omega, mode, n_iter, tol, K, measure_last) -> Report:
    f64 = u.dtype == np.float64
    _grid(u, np.float64 if f64 else np.float32)
    r = _Report()
    fn = lib().orc_variant_run_f64 if f64 else lib().orc_variant_run_f32
    fn(u.ctypes.data, u.shape[0] - 2, u.shape[1] - 2, kind, p1, p2, p3, omega, mode, n_iter, tol, K,
       int(measure_last), ctypes.byref(r))
    if r.status < 0:
        raise ValueError("oracle rejected arguments")
    return _rep(r)


def multicolor_iterate(u: np.ndarray, omega: float, iters: int, ca: int = 1, cb: int = 1, nc: int = 2,
                       measure_last: bool = False) -> Report:
    """NEXT-4 (reading N4-1): multi-colour SOR, colour (ca*i + cb*j) mod nc, phases 0..nc-1."""
    return _variant(u, 0, ca, cb, nc, omega, 0, iters, 1.0, 1, measure_last)


def multicolor_solve(u: np.ndarray, omega: float, tol: float, maxit: int, check_every: int = 1,
                     ca: int = 1, cb: int = 1, nc: int = 2) -> Report:
    return _variant(u, 0, ca, cb, nc, omega, 1, maxit, tol, check_every, False)


def block_iterate(u: np.ndarray, omega: float, iters: int, block: int, measure_last: bool = False) -> Report:
    """NEXT-4 (reading N4-2): block red-black SOR, natural order inside block x block blocks."""
    return _variant(u, 1, block, 0, 0, omega, 0, iters, 1.0, 1, measure_last)


def block_solve(u: np.ndarray, omega: float, tol: float, maxit: int, block: int, check_every: int = 1) -> Report:
    return _variant(u, 1, block, 0, 0, omega, 1, maxit, tol, check_every, False)


def dense_solve3d(u: np.ndarray) -> None:
    assert u.ndim == 3 and u.dtype == np.float64 and u.flags.c_contiguous
    if lib().orc_dense_solve3d_f64(u.ctypes.data, u.shape[0] - 2, u.shape[1] - 2, u.shape[2] - 2) != 0:
        raise ValueError("dense 3-D solve limited to 1728 unknowns")


def dense_solve(u: np.ndarray) -> None:
    _grid(u, np.float64)
    if lib().orc_dense_solve_f64(u.ctypes.data, u.shape[0] - 2, u.shape[1] - 2) != 0:
        raise ValueError("dense solve limited to rows*cols <= 4096")


def cell_update(n, s, w, e, u, omega, dtype="f64"):
    if dtype == "f64":
        return lib().orc_cell_update_f64(n, s, w, e, u, omega)
    return lib().orc_cell_update_f32(n, s, w, e, u, omega)
