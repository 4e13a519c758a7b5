"""C-ABI contract checks that need no GPU (`-m "not gpu"`).

The library must build, load and export every symbol include/sor.h declares;
argument validation happens before any device work; without a GPU the
create calls fail loudly (no CPU fallback).
"""
import ctypes
import os
import re

import pytest

import paper_1401_0763_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "sor.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sor(?:3d)?_[a-z0-9_]+)\s*\(", src)))


def _gpu_present():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_library_builds_and_exports_every_declared_symbol():
    L = P.lib()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(P.EXPORTS)


def test_sm100a_only_binary():
    out = os.popen(f"cuobjdump --list-elf {P.LIB} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_partition_rows_host_logic(orc):
    for rows in (8, 9, 100, 4096, 32768 * 8 + 3):
        for nparts in (1, 2, 3, 4, 8):
            spans = [P.partition_rows(rows, nparts, p) for p in range(nparts)]
            assert spans[0][0] == 1 and spans[-1][1] == rows + 1
            assert all(spans[p][1] == spans[p + 1][0] for p in range(nparts - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
            # independent implementation in the oracle agrees
            assert spans == [orc.partition_rows(rows, nparts, p) for p in range(nparts)]
    with pytest.raises(P.SorError):
        P.partition_rows(3, 4, 0)
    with pytest.raises(P.SorError):
        P.partition_rows(10, 2, 2)


def test_validation_before_device_work():
    L = P.lib()
    h = ctypes.c_void_p()
    import numpy as np
    a = np.zeros((6, 6))
    assert L.sor_create(None, 4, a.ctypes.data, 0) == P.SOR_E_INVAL
    assert L.sor_create(ctypes.byref(h), 4, None, 0) == P.SOR_E_INVAL
    assert L.sor_create(ctypes.byref(h), 0, a.ctypes.data, 0) == P.SOR_E_INVAL
    assert L.sor_create_rect(ctypes.byref(h), 4, -1, a.ctypes.data, 0) == P.SOR_E_INVAL
    assert L.sor_create(ctypes.byref(h), 4, a.ctypes.data, 7) == P.SOR_E_INVAL
    assert "dtype" in P.last_error()
    assert L.sor_create_virtual(ctypes.byref(h), 4, 4, a.ctypes.data, 0, 2) == P.SOR_E_INVAL
    assert L.sor_iterate(None, 1.5, 3, None) == P.SOR_E_INVAL
    assert L.sor_solve(None, 1.5, 1e-3, 10, 1, None, None) == P.SOR_E_INVAL
    assert L.sor_download(None, None) == P.SOR_E_INVAL
    d = ctypes.c_double()
    assert L.sor_last_elapsed_ms(None, ctypes.byref(d)) == P.SOR_E_INVAL
    L.sor_destroy(None)   # NULL-safe


@pytest.mark.skipif(_gpu_present(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    import numpy as np
    a = np.zeros((6, 6))
    h = ctypes.c_void_p()
    rc = P.lib().sor_create(ctypes.byref(h), 4, a.ctypes.data, 0)
    assert rc == P.SOR_E_CUDA
    assert "no CPU fallback" in P.last_error() or "CUDA" in P.last_error()
    with pytest.raises(P.SorError):
        P.Grid.create(a)


def test_python_binding_has_no_compute():
    """The binding is marshalling only: no numpy arithmetic on grid values."""
    src = open(os.path.join(ROOT, "paper_1401_0763_b200", "__init__.py")).read()
    assert "import oracle" not in src and "from oracle" not in src
    for bad in ("0.25", "omega *", "* omega", ".max(", "np.abs("):
        assert bad not in src, bad


def test_device_copies_are_stream_ordered():
    """Every host->device copy and memset in the C-ABI runs on the grid's own
    (non-blocking) stream: a legacy-stream cudaMemcpy/cudaMemset is not ordered
    with the kernels and, from pageable memory, may return before the DMA lands."""
    import re
    import glob
    src = "".join(open(f).read() for f in glob.glob(os.path.join(ROOT, "paper_1401_0763_b200", "csrc", "*.cu")))
    assert not re.findall(r"\bcudaMemcpy(?:2D)?\(", src)
    assert not re.findall(r"\bcudaMemset\(", src)


def test_binding_rejects_wrong_buffers_before_the_c_call():
    """The binding checks dtype, contiguity and the exact shape of every grid
    buffer before handing a raw pointer to C (a wrong size there is an
    out-of-bounds access), and maps dtype names explicitly."""
    import numpy as np
    good = np.zeros((6, 9))
    assert P._ptr(good, shape=(6, 9))[0] == good.ctypes.data
    with pytest.raises(ValueError):
        P._ptr(good, shape=(9, 6))
    with pytest.raises(ValueError):
        P._ptr(np.zeros(54), shape=(6, 9))
    with pytest.raises(TypeError):
        P._ptr(np.zeros((6, 9), dtype=np.float32), shape=(6, 9))
    with pytest.raises(TypeError):
        P._ptr(np.zeros((9, 6)).T, shape=(6, 9))            # not C-contiguous
    ro = np.zeros((6, 9))
    ro.flags.writeable = False
    with pytest.raises(TypeError):
        P._ptr(ro, writable=True, shape=(6, 9))
    with pytest.raises(TypeError):
        P._ptr([[0.0] * 9] * 6, shape=(6, 9))
    import torch
    t = torch.zeros(6, 9, dtype=torch.float64)
    assert P._ptr(t, shape=(6, 9))[0] == t.data_ptr()
    with pytest.raises(ValueError):
        P._ptr(t, shape=(6, 8))
    with pytest.raises(TypeError):
        P._ptr(t.float(), shape=(6, 9))
    assert P._dt("f64") == P.F64 and P._dt("f32") == P.F32
    for bad in ("float64", "fp64", "F64", "", None):
        with pytest.raises(ValueError):
            P._dt(bad)
    with pytest.raises(ValueError):
        P.Grid.create(np.zeros((6, 9)), dtype="double")
    with pytest.raises(ValueError):
        P.Grid.create(np.zeros(54))
