"""Build libskb200.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2301_03598_b200.build        # or __graft_entry__.build()

The shared library links the CUDA runtime statically and libstdc++ statically,
and exports only the sk_* C symbols (csrc/exports.map), so it loads next to
torch / numpy without symbol clashes.  The driver API (cuTensorMapEncodeTiled)
is reached through cudaGetDriverEntryPoint, so no -lcuda is needed to link.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libskb200.so")

SOURCES = ["skb200_api.cu", "sk_gemm_f16.cu", "sk_gemm_f64.cu", "sk_convert.cu", "sk_random.cu",
           "sk_probe.cu", "costmodel.cpp", "skmx.cpp", "simulate.cpp"]
HEADERS = ["ptx.cuh", "schedule.hpp", "sk_kernel_common.cuh", "exports.map"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "skb200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str = "") -> str:
    """Build libskb200.so; `out` (or $SKB200_LIB_OUT) writes an experimental
    variant elsewhere (loaded with $SKB200_LIB) instead of the product library."""
    out = out or os.environ.get("SKB200_LIB_OUT", "")
    lib = out or LIB
    if not out and not force and not _stale():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    tmp = lib + ".tmp"
    cmd = [
        nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
        "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
        "-Xlinker", "--version-script=" + os.path.join(CSRC, "exports.map"),
        "-Xcompiler", "-static-libstdc++", "-Xcompiler", "-static-libgcc",
        "-cudart", "static",
        *os.environ.get("SKB200_DEFINES", "").split(),
        *[os.path.join(CSRC, f) for f in SOURCES],
        "-o", tmp,
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc build of libskb200.so failed")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
