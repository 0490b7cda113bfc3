"""Build libcrsh.so in-tree: nvcc for sm_100a only (no other arch, no JIT).

Numeric flags: --fmad=false (no implicit contraction; the
kernels use explicit __fmaf_rn where NUMSPEC says fma), IEEE division and
square root, no flush-to-zero, never --use_fast_math."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "crsh.cu")
OUT = os.path.join(HERE, "libcrsh.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "--fmad=false",
         "-prec-div=true", "-prec-sqrt=true", "-ftz=false", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static"]


def nccl_dir() -> str:
    """The NCCL 2.28 that torch ships (headers incl. the device API, and
    libnccl.so.2); libcrsh links it with an rpath, so a process that already
    loaded torch's NCCL shares that one copy (same soname)."""
    import nvidia.nccl
    return list(nvidia.nccl.__path__)[0]


def nccl_flags():
    d = nccl_dir()
    return ["-I" + os.path.join(d, "include"), "-L" + os.path.join(d, "lib"), "-l:libnccl.so.2", "-Xlinker",
            "-rpath=" + os.path.join(d, "lib")]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu*"))) + [os.path.join(os.path.dirname(HERE), "include",
                                                                                 "crsh.h")]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        cmd = [NVCC, *FLAGS, *nccl_flags(), *(["-Xptxas", "-v"] if verbose else []), "-o", OUT + ".tmp", SRC]
        subprocess.check_call(cmd)
        os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(force=True, verbose=True)
