"""Build librmx.so (the C-ABI library, include/rmx.h) in-tree with nvcc for sm_100a.

    python -m paper_1403_5524_b200.build [--force]

nvcc cross-compiles without a GPU, so this runs on the CPU build box as well.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "librmx.so")
SOURCES = ["rform.cu", "rint8.cu", "match.cu", "tepi.cu", "photo.cu", "post.cu", "rmx_api.cu"]
HEADERS = ["rmx_common.cuh", "cta_la.cuh", "rmx_internal.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared"]
# cuSOLVER (syevd) + cuBLAS (one DGEMM) serve only the inner-region eigensolve (NEXT-3)
LIBS = ["-L/usr/local/cuda/lib64", "-lcusolver", "-lcublas", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(PKG), "include", "rmx.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_phases(verbose: bool = False, suffix: str = "", defines=()) -> str:
    """Diagnostic variant with per-phase clock64 counters in the matching kernel (librmx_phases.so);
    suffix/defines build A/B variants (librmx_phases<suffix>.so with extra -D flags)."""
    out = os.path.join(PKG, f"librmx_phases{suffix}.so")
    cmd = [NVCC, *FLAGS, "-DRMX_PHASES", *[f"-D{d}" for d in defines], "-o", out,
           *[os.path.join(CSRC, s) for s in SOURCES], *LIBS]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=CSRC)
    return out


def build_variant(suffix: str, defines=(), verbose: bool = False) -> str:
    """A/B variant of the product library (librmx_<suffix>.so with extra -D flags), selected at run
    time with RMX_LIB=... (e.g. RMX_NO_TILE_PAIRS: the row-major tile order everywhere)."""
    out = os.path.join(PKG, f"librmx_{suffix}.so")
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out, *[os.path.join(CSRC, s) for s in SOURCES], *LIBS]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=CSRC)
    return out


def build_checked(force: bool = False, verbose: bool = False) -> str:
    """Bounds-checked variant (librmx_checked.so, -DRMX_CHECKS): device-side index / extent checks
    that trap (rmx_common.cuh RMX_CHECK) - the stand-in for compute-sanitizer, which is closed on
    the GPU pool (tests/test_gpu_checked.py)."""
    out = os.path.join(PKG, "librmx_checked.so")
    if not force and os.path.exists(out) and not _stale(out):
        return out
    cmd = [NVCC, *FLAGS, "-DRMX_CHECKS", "-o", out, *[os.path.join(CSRC, s) for s in SOURCES], *LIBS]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=CSRC)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES], *LIBS]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    if "--phases" in sys.argv:
        # --phases [SUFFIX DEFINE ...]: an A/B variant of the diagnostic build
        rest = sys.argv[sys.argv.index("--phases") + 1:]
        print(build_phases(verbose=True, suffix=rest[0] if rest else "", defines=rest[1:]))
    elif "--checked" in sys.argv:
        print(build_checked(force=True, verbose=True))
    else:
        build(force="--force" in sys.argv, verbose=True)
        print(LIB)
