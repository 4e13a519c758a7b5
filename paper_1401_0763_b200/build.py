"""Build libsor.so in-tree with nvcc for sm_100a (B200).

The library is the product: C ABI in include/sor.h, kernels in csrc/.  It
links NCCL 2.28 from the torch wheel (nvidia/nccl) for the multi-GPU path.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libsor.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no FMA contraction (reading #4); FTZ stays off (reading #17).
# (--split-compile halves the build time but changed the wave kernel's SASS
# and cost 1.3% at C3/C5, so it is not used.)
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-fmad=false", "-ftz=false", "-prec-div=true",
              "-prec-sqrt=true", "-Xcompiler", "-fPIC", "-shared", *ARCH]


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


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(INCLUDE, "sor.h")])


def build_lib(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    stale = not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(s) for s in sources())
    if not (force or stale):
        return out
    nc = nccl_dir()
    cmd = [NVCC, *NVCC_FLAGS, *("-D" + d for d in defines), "-I" + INCLUDE, "-I" + os.path.join(nc, "include"),
           os.path.join(CSRC, "sor_api.cu"), "-o", out + ".tmp",
           "-L" + os.path.join(nc, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nc, "lib")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build_lib(force=True, verbose=True))
