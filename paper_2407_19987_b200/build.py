"""Compile the CUDA library in-tree: paper_2407_19987_b200/_lib/libhobo.so (sm_100a only)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libhobo.so")
SOURCES = [os.path.join(CSRC, f) for f in ("hobo_api.cu", "host_compile.cpp", "tt.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("kernels.cuh", "ptx.cuh", "host_compile.h", "tt.h")] + [
    os.path.join(ROOT, "include", "hobo.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",  # tcgen05 needs the arch-specific target
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
    "-I" + os.path.join(ROOT, "include"),
]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, debug_stats: bool = False) -> str:
    """debug_stats=True builds _lib/libhobo_dbg.so with per-CTA pipeline counters (tools only)."""
    lib = LIB.replace("libhobo.so", "libhobo_dbg.so") if debug_stats else LIB
    if not force and not debug_stats and not stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    cmd = [NVCC, *FLAGS, *(["-DHOBO_PIPE_STATS"] if debug_stats else []), *(["-Xptxas", "-v"] if verbose else []),
           "-o", lib, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libhobo.so")
    if verbose:
        sys.stderr.write(r.stderr)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug_stats="--debug-stats" in sys.argv))
