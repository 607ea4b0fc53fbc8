"""Build libozaki.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libozaki.so")
SHIM = os.path.join(PKG, "libozaki_blas.so")   # Fortran dgemm_/zgemm_ interposition (NEXT-2)
SOURCES = ["ozaki.cu"]
HEADERS = ["split_cluster.cuh", "trsm.cuh", "crt.cuh", "crt_kernel.cuh", "gemm_crt.cuh", "gemm_lv2.cuh", "passplan.cuh", "gemm_lv.cuh", "gemm.cuh", "split.cuh", "split_fast.cuh", "numerics.cuh", "ptx.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "ozaki.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build_shim(force: bool = False) -> str:
    """libozaki_blas.so: dgemm_/zgemm_ (Fortran ABI) -> libozaki.so, rpath $ORIGIN."""
    src = os.path.join(CSRC, "blas_shim.cpp")
    deps = [src, os.path.join(ROOT, "include", "ozaki.h"), LIB]
    if not force and os.path.exists(SHIM) and all(os.path.getmtime(d) <= os.path.getmtime(SHIM) for d in deps):
        return SHIM
    tmp = SHIM + f".tmp{os.getpid()}"
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-I", os.path.join(ROOT, "include"),
           src, "-o", tmp, "-L", PKG, "-l:libozaki.so", "-Wl,-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("building libozaki_blas.so failed")
    os.replace(tmp, SHIM)
    return SHIM


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        build_shim()
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, LIB)
    build_shim(force=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
