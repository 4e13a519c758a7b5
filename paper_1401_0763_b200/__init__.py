"""B200-native red-black SOR hot path (arXiv 1401.0763) — Python binding.

Thin ctypes marshalling over libsor.so (C ABI: include/sor.h).  Every step
of the method runs in the library's CUDA kernels; this module only passes
pointers and sizes.  There is no CPU fallback: if libsor.so is missing or no
B200 is visible, the calls raise.

Arrays are the full (rows+2) x (cols+2) fp64 grid including the Dirichlet
ring (row 0 = north), given as a C-contiguous numpy float64 array or a
contiguous torch float64 tensor on the host or on the handle's GPU.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from .build import LIB, build_lib

SOR_OK, SOR_NOT_CONVERGED = 0, 1
SOR_E_INVAL, SOR_E_NOMEM, SOR_E_CUDA, SOR_E_NCCL, SOR_E_STATE, SOR_E_UNSUPPORTED = -1, -2, -3, -4, -5, -6
F64, F32 = 0, 1
KERNEL_NATURAL, KERNEL_FUSED, KERNEL_TEMPORAL, KERNEL_SMALL, KERNEL_RESIDENT = 1, 3, 4, 5, 6
KERNELS = {"natural": KERNEL_NATURAL, "k1": KERNEL_NATURAL, "fused": KERNEL_FUSED, "k3": KERNEL_FUSED,
           "temporal": KERNEL_TEMPORAL, "k4": KERNEL_TEMPORAL, "small": KERNEL_SMALL, "k5": KERNEL_SMALL,
           "resident": KERNEL_RESIDENT, "k7": KERNEL_RESIDENT}

EXPORTS = ("sor_create", "sor_create_rect", "sor_create_dist", "sor_nccl_unique_id",
           "sor_create_dist_ipc", "sor_ipc_unique_id",
           "sor_create_virtual", "sor_set_kernel", "sor_iterate", "sor_solve", "sor_download",
           "sor_download_rows", "sor_reset", "sor_set_stream", "sor_last_elapsed_ms", "sor_get_stats",
           "sor_partition_rows", "sor_destroy", "sor_last_error", "sor_jacobi_iterate", "sor_jacobi_solve",
           "sor3d_create", "sor3d_iterate", "sor3d_solve", "sor3d_download", "sor3d_last_elapsed_ms",
           "sor3d_destroy", "sor3d_set_kernel", "sor_variant_iterate", "sor_variant_solve")
VARIANT_MULTICOLOR, VARIANT_BLOCK = 1, 2


class Variant(ctypes.Structure):
    """sor_variant (include/sor.h): NEXT-4 multi-colour / block red-black SOR."""
    _fields_ = [("kind", ctypes.c_int32), ("ca", ctypes.c_int32), ("cb", ctypes.c_int32),
                ("nc", ctypes.c_int32), ("block", ctypes.c_int32)]

    @classmethod
    def multicolor(cls, ca: int = 1, cb: int = 1, nc: int = 2) -> "Variant":
        return cls(VARIANT_MULTICOLOR, ca, cb, nc, 0)

    @classmethod
    def blocks(cls, block: int) -> "Variant":
        return cls(VARIANT_BLOCK, 0, 0, 0, block)


class SorError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("half_sweeps", ctypes.c_int64),
                ("halo_exchanges", ctypes.c_int64), ("checks", ctypes.c_int64),
                ("hbm_passes", ctypes.c_int64), ("kernel", ctypes.c_int32),
                ("temporal_depth", ctypes.c_int32), ("nslabs", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("row_lo", ctypes.c_int64), ("row_hi", ctypes.c_int64),
                ("pitch_elems", ctypes.c_int64), ("exact_reruns", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load libsor.so (building it with nvcc if absent and allowed)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SOR_LIBRARY", LIB)   # development: alternative builds of libsor
    if not os.path.exists(path):
        if not build_if_missing:
            raise FileNotFoundError(f"{path} not built; run __graft_entry__.build()")
        build_lib()
    L = ctypes.CDLL(path)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    pp = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "sor_create": (i32, [pp, i64, vp, i32]),
        "sor_create_rect": (i32, [pp, i64, i64, vp, i32]),
        "sor_create_dist": (i32, [pp, i64, i64, vp, i32, i32, i32, i32, vp]),
        "sor_nccl_unique_id": (i32, [vp]),
        "sor_create_dist_ipc": (i32, [pp, i64, i64, vp, i32, i32, i32, i32, vp]),
        "sor_ipc_unique_id": (i32, [vp]),
        "sor_create_virtual": (i32, [pp, i64, i64, vp, i32, i32]),
        "sor_set_kernel": (i32, [vp, i32, i32]),
        "sor_iterate": (i32, [vp, dbl, i64, ctypes.POINTER(dbl)]),
        "sor_solve": (i32, [vp, dbl, dbl, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(dbl)]),
        "sor_download": (i32, [vp, vp]),
        "sor_jacobi_iterate": (i32, [vp, i64, ctypes.POINTER(dbl)]),
        "sor_jacobi_solve": (i32, [vp, dbl, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(dbl)]),
        "sor_download_rows": (i32, [vp, i64, i64, vp]),
        "sor_reset": (i32, [vp, vp]),
        "sor_set_stream": (i32, [vp, vp]),
        "sor_last_elapsed_ms": (i32, [vp, ctypes.POINTER(dbl)]),
        "sor_get_stats": (i32, [vp, ctypes.POINTER(Stats)]),
        "sor_partition_rows": (i32, [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "sor_destroy": (None, [vp]),
        "sor3d_create": (i32, [pp, i64, i64, i64, vp, i32]),
        "sor3d_iterate": (i32, [vp, dbl, i64, ctypes.POINTER(dbl)]),
        "sor3d_solve": (i32, [vp, dbl, dbl, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(dbl)]),
        "sor3d_download": (i32, [vp, vp]),
        "sor3d_last_elapsed_ms": (i32, [vp, ctypes.POINTER(dbl)]),
        "sor3d_destroy": (None, [vp]),
        "sor3d_set_kernel": (i32, [vp, i32]),
        "sor_variant_iterate": (i32, [vp, ctypes.POINTER(Variant), dbl, i64, ctypes.POINTER(dbl)]),
        "sor_variant_solve": (i32, [vp, ctypes.POINTER(Variant), dbl, dbl, i64, i64, ctypes.POINTER(i64),
                                    ctypes.POINTER(dbl)]),
        "sor_last_error": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def last_error() -> str:
    return lib().sor_last_error().decode()


def _check(rc: int, allow_not_converged: bool = False) -> int:
    if rc < 0 or (rc == SOR_NOT_CONVERGED and not allow_not_converged):
        raise SorError(rc, last_error())
    return rc


def _ptr(a, writable: bool = False, shape=None):
    """(address, keepalive) of a float64 grid buffer (numpy or torch), after
    checking dtype, contiguity and (if given) the exact shape the C call will
    read or write: a wrong size would be an out-of-bounds access in C."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise TypeError("grid must be a C-contiguous float64 array")
        if writable and not a.flags.writeable:
            raise TypeError("output array is read-only")
        if shape is not None and tuple(a.shape) != tuple(shape):
            raise ValueError(f"buffer shape {tuple(a.shape)} != expected {tuple(shape)}")
        return a.ctypes.data, a
    if hasattr(a, "data_ptr"):  # torch.Tensor
        import torch
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise TypeError("grid tensor must be contiguous float64")
        if shape is not None and tuple(a.shape) != tuple(shape):
            raise ValueError(f"buffer shape {tuple(a.shape)} != expected {tuple(shape)}")
        return a.data_ptr(), a
    raise TypeError(f"unsupported grid buffer {type(a)!r}")


_DTYPES = {"f64": F64, "f32": F32}


def _dt(dtype: str) -> int:
    try:
        return _DTYPES[dtype]
    except KeyError:
        raise ValueError(f"dtype must be 'f64' or 'f32', got {dtype!r}") from None


def partition_rows(rows: int, P: int, p: int) -> tuple[int, int]:
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().sor_partition_rows(rows, P, p, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().sor_nccl_unique_id(buf))
    return buf.raw


def ipc_unique_id() -> bytes:
    """Rendezvous id of a dist-IPC handle (rank 0 makes it; broadcast it)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().sor_ipc_unique_id(buf))
    return buf.raw


@dataclass
class SolveResult:
    converged: bool
    iters: int
    max_change: float


class Grid:
    """A device-resident SOR grid (one handle of libsor.so)."""

    def __init__(self, handle: int, rows: int, cols: int, dtype: str):
        self._h = ctypes.c_void_p(handle)
        self.rows, self.cols, self.dtype = rows, cols, dtype

    # ---- construction
    @classmethod
    def create(cls, init, dtype: str = "f64", rows: int | None = None, cols: int | None = None):
        rows, cols = cls._dims(init, rows, cols)
        h = ctypes.c_void_p()
        p, _keep = _ptr(init, shape=(rows + 2, cols + 2))
        _check(lib().sor_create_rect(ctypes.byref(h), rows, cols, p, _dt(dtype)))
        return cls(h.value, rows, cols, dtype)

    @classmethod
    def create_virtual(cls, init, nslabs: int, dtype: str = "f64"):
        rows, cols = cls._dims(init, None, None)
        h = ctypes.c_void_p()
        p, _keep = _ptr(init, shape=(rows + 2, cols + 2))
        _check(lib().sor_create_virtual(ctypes.byref(h), rows, cols, p, _dt(dtype), nslabs))
        return cls(h.value, rows, cols, dtype)

    @classmethod
    def _create_dist(cls, fn, init, rank, nranks, device, uid, dtype, rows, cols):
        if init is None:
            if rows is None or cols is None:
                raise ValueError("init=None needs rows and cols")
            p, _keep = None, None
        else:
            rows, cols = cls._dims(init, rows, cols)
            p, _keep = _ptr(init, shape=(rows + 2, cols + 2))
        h = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(bytes(uid), 128)
        _check(fn(ctypes.byref(h), rows, cols, p, _dt(dtype), rank, nranks, device, idbuf))
        g = cls(h.value, rows, cols, dtype)
        g.rank, g.nranks = rank, nranks
        return g

    @classmethod
    def create_dist(cls, init, rank: int, nranks: int, device: int, nccl_id: bytes,
                    dtype: str = "f64", rows: int | None = None, cols: int | None = None):
        """Dist handle over NCCL (fallback transport); init only on rank 0."""
        return cls._create_dist(lib().sor_create_dist, init, rank, nranks, device, nccl_id, dtype, rows, cols)

    @classmethod
    def create_dist_ipc(cls, init, rank: int, nranks: int, device: int, ipc_id: bytes,
                        dtype: str = "f64", rows: int | None = None, cols: int | None = None):
        """Dist handle over CUDA IPC (device-initiated halo push); init only on rank 0."""
        return cls._create_dist(lib().sor_create_dist_ipc, init, rank, nranks, device, ipc_id, dtype, rows, cols)

    @staticmethod
    def _dims(init, rows, cols):
        shape = tuple(init.shape)
        if len(shape) != 2:
            raise ValueError("init must be 2-D (rows+2, cols+2)")
        r, c = shape[0] - 2, shape[1] - 2
        if (rows is not None and rows != r) or (cols is not None and cols != c):
            raise ValueError("rows/cols do not match init shape")
        return r, c

    # ---- configuration
    def set_kernel(self, kernel, temporal_depth: int = 1) -> "Grid":
        k = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
        _check(lib().sor_set_kernel(self._h, k, temporal_depth))
        return self

    def set_stream(self, stream_ptr: int | None) -> None:
        _check(lib().sor_set_stream(self._h, ctypes.c_void_p(stream_ptr or 0)))

    # ---- the hot path
    def iterate(self, omega: float, iters: int, want_delta: bool = False):
        d = ctypes.c_double(0.0)
        _check(lib().sor_iterate(self._h, omega, iters, ctypes.byref(d) if want_delta else None))
        return d.value if want_delta else None

    def solve(self, omega: float, tol: float, maxit: int, check_every: int = 1) -> SolveResult:
        it, m = ctypes.c_int64(0), ctypes.c_double(0.0)
        rc = _check(lib().sor_solve(self._h, omega, tol, maxit, check_every, ctypes.byref(it),
                                    ctypes.byref(m)), allow_not_converged=True)
        return SolveResult(rc == SOR_OK, it.value, m.value)

    def jacobi(self, iters: int, want_delta: bool = False):
        """NEXT-2: `iters` Jacobi iterations on the device."""
        d = ctypes.c_double(0.0)
        _check(lib().sor_jacobi_iterate(self._h, iters, ctypes.byref(d) if want_delta else None))
        return d.value if want_delta else None

    def jacobi_solve(self, tol: float, maxit: int, check_every: int = 1) -> SolveResult:
        it, m = ctypes.c_int64(0), ctypes.c_double(0.0)
        rc = _check(lib().sor_jacobi_solve(self._h, tol, maxit, check_every, ctypes.byref(it), ctypes.byref(m)),
                    allow_not_converged=True)
        return SolveResult(rc == SOR_OK, it.value, m.value)

    def variant_iterate(self, variant: "Variant", omega: float, iters: int, want_delta: bool = False):
        """NEXT-4: `iters` iterations of a multi-colour / block SOR variant."""
        d = ctypes.c_double()
        _check(lib().sor_variant_iterate(self._h, ctypes.byref(variant), omega, iters,
                                         ctypes.byref(d) if want_delta else None))
        return d.value if want_delta else None

    def variant_solve(self, variant: "Variant", omega: float, tol: float, maxit: int,
                      check_every: int = 1) -> SolveResult:
        it, m = ctypes.c_int64(0), ctypes.c_double(0.0)
        rc = _check(lib().sor_variant_solve(self._h, ctypes.byref(variant), omega, tol, maxit, check_every,
                                            ctypes.byref(it), ctypes.byref(m)), allow_not_converged=True)
        return SolveResult(rc == SOR_OK, it.value, m.value)

    def _receives(self) -> bool:
        return getattr(self, "rank", 0) == 0

    def download(self, out=None):
        """The whole grid; dist handles: collective, rank 0 receives (others get None)."""
        if not self._receives():
            _check(lib().sor_download(self._h, None))
            return None
        if out is None:
            out = np.empty((self.rows + 2, self.cols + 2), dtype=np.float64)
        p, _keep = _ptr(out, writable=True, shape=(self.rows + 2, self.cols + 2))
        _check(lib().sor_download(self._h, p))
        return out

    def download_rank_nonzero(self):
        """Dist ranks != 0 participate in the gather without a buffer."""
        _check(lib().sor_download(self._h, None))

    def download_rows(self, row_a: int, row_b: int, out=None):
        """Global rows [row_a, row_b) (ring rows count: 0 is the north ring).
        Dist handles: collective, rank 0 receives (others get None)."""
        if not self._receives():
            _check(lib().sor_download_rows(self._h, row_a, row_b, None))
            return None
        if out is None:
            out = np.empty((max(0, row_b - row_a), self.cols + 2), dtype=np.float64)
        p, _keep = _ptr(out, writable=True, shape=(max(0, row_b - row_a), self.cols + 2))
        _check(lib().sor_download_rows(self._h, row_a, row_b, p))
        return out

    def reset(self, init) -> None:
        """Reload from init (dist: collective; init read on rank 0, None elsewhere)."""
        if init is None:
            _check(lib().sor_reset(self._h, None))
            return
        p, _keep = _ptr(init, shape=(self.rows + 2, self.cols + 2))
        _check(lib().sor_reset(self._h, p))

    @property
    def elapsed_ms(self) -> float:
        d = ctypes.c_double()
        _check(lib().sor_last_elapsed_ms(self._h, ctypes.byref(d)))
        return d.value

    @property
    def stats(self) -> dict:
        s = Stats()
        _check(lib().sor_get_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def close(self) -> None:
        if self._h is not None and self._h.value:
            lib().sor_destroy(self._h)
        self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Grid3D:
    """NEXT-3: a device-resident 3-D red-black SOR grid (sor3d_* handle).
    Arrays are (nz+2, ny+2, nx+2) C-contiguous fp64 (numpy or torch)."""

    def __init__(self, init, dtype: str = "f64"):
        if len(tuple(init.shape)) != 3:
            raise ValueError("init must be 3-D (nz+2, ny+2, nx+2)")
        self.nz, self.ny, self.nx = (int(d) - 2 for d in init.shape)
        self.dtype = dtype
        h = ctypes.c_void_p()
        p, _keep = _ptr(init)
        _check(lib().sor3d_create(ctypes.byref(h), self.nz, self.ny, self.nx, p, _dt(dtype)))
        self._h = h

    def set_kernel(self, kernel) -> "Grid3D":
        k = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
        _check(lib().sor3d_set_kernel(self._h, k))
        return self

    def iterate(self, omega: float, iters: int, want_delta: bool = False):
        d = ctypes.c_double(0.0)
        _check(lib().sor3d_iterate(self._h, omega, iters, ctypes.byref(d) if want_delta else None))
        return d.value if want_delta else None

    def solve(self, omega: float, tol: float, maxit: int, check_every: int = 1) -> SolveResult:
        it, m = ctypes.c_int64(0), ctypes.c_double(0.0)
        rc = _check(lib().sor3d_solve(self._h, omega, tol, maxit, check_every, ctypes.byref(it), ctypes.byref(m)),
                    allow_not_converged=True)
        return SolveResult(rc == SOR_OK, it.value, m.value)

    def download(self, out=None):
        shape = (self.nz + 2, self.ny + 2, self.nx + 2)
        if out is None:
            out = np.empty(shape, dtype=np.float64)
        p, _keep = _ptr(out, writable=True, shape=shape)
        _check(lib().sor3d_download(self._h, p))
        return out

    @property
    def elapsed_ms(self) -> float:
        d = ctypes.c_double()
        _check(lib().sor3d_last_elapsed_ms(self._h, ctypes.byref(d)))
        return d.value

    def close(self) -> None:
        if self._h is not None and self._h.value:
            lib().sor3d_destroy(self._h)
        self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
