"""Build libsor.so in-tree with nvcc for sm_100a (B200).

The library is the product: C ABI in include/sor.h, kernels in csrc/.  It
links NCCL 2.28 from the torch wheel (nvidia/nccl) for the NCCL transport
of the multi-GPU path.  The translation units (driver, one per kernel
family / depth) compile in parallel, then link into one shared object.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libsor.so")
OBJDIR = os.path.join(os.environ.get("SORB_OBJDIR", "/tmp"), "sorb_build_obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no FMA contraction (reading #4); FTZ stays off (reading #17).
# (--split-compile changed the wave kernel's SASS and cost 1.3% at C3/C5, so
# the parallelism comes from separate translation units instead.)
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-fmad=false", "-ftz=false", "-prec-div=true",
              "-prec-sqrt=true", "-Xcompiler", "-fPIC", *ARCH]


def nccl_dir() -> str:
    cands = [os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")]
    try:
        import nvidia  # noqa: F401
        for p in getattr(__import__("nvidia"), "__path__", []):
            cands.append(os.path.join(p, "nccl"))
    except Exception:
        pass
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("NCCL headers not found (expected the torch wheel's nvidia/nccl)")


def units() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def sources() -> list[str]:
    return sorted(units() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + [os.path.join(INCLUDE, "sor.h")])


def build_lib(force: bool = False, verbose: bool = False, out: str = LIB, defines=(), jobs: int | None = None) -> str:
    stale = not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(s) for s in sources())
    if not (force or stale):
        return out
    nc = nccl_dir()
    tag = "".join(d.replace("=", "_") for d in defines)
    objdir = OBJDIR + (("_" + tag) if tag else "")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I" + INCLUDE, "-I" + os.path.join(nc, "include")]
    dflags = ["-D" + d for d in defines]

    hdr_mtime = max(os.path.getmtime(h) for h in sources() if not h.endswith(".cu"))

    def compile_one(src: str) -> str:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        # incremental (not forced): a unit is rebuilt if it or any header is newer than its object
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_mtime)):
            return obj
        cmd = [NVCC, *NVCC_FLAGS, *dflags, *inc, "-c", src, "-o", obj + ".tmp"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        os.replace(obj + ".tmp", obj)
        return obj

    jobs = jobs or max(1, min(len(units()), os.cpu_count() or 4))
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        # longest units first
        srcs = sorted(units(), key=lambda s: (not os.path.basename(s).startswith("wave_"), s))
        objs = list(ex.map(compile_one, srcs))
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", out + ".tmp",
           "-L" + os.path.join(nc, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nc, "lib"), "-lrt"]
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import sys
    print(build_lib(force=True, verbose="-v" in sys.argv))
