"""Build the in-tree CUDA library libsphbuf.so for sm_100a (nvcc, no GPU needed)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libsphbuf.so")
LIB_DEBUG = os.path.join(HERE, "libsphbuf_debug.so")   # -DSPHBUF_DEBUG: device bounds asserts
LIB_TRACE = os.path.join(HERE, "libsphbuf_trace.so")   # -DSPHBUF_TRACE: per-tile timestamps of the update (tools/)
SOURCES = ["sphbuf_cll.cu", "sphbuf_update.cu", "sphbuf_compact.cu", "sphbuf_migrate.cu", "sphbuf_motion.cu",
           "sphbuf_drivers.cu", "sphbuf_host.cpp", "sphbuf_comm.cpp"]
DEPS = SOURCES + ["sphbuf_internal.h", "sphbuf_common.cuh", "sphbuf_tma.cuh", "sphbuf_prologue.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "--fmad=false",
         "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared", "-Xptxas", "-v"]


def _stale(lib=LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    srcs = [os.path.join(CSRC, s) for s in DEPS] + [os.path.join(INCLUDE, "sphbuf.h")]
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False, debug: bool = False, trace: bool = False) -> str:
    """Compile libsphbuf.so (or, debug=True, libsphbuf_debug.so with device-side
    bounds asserts: compute-sanitizer is not available on the GPU pool; or,
    trace=True, libsphbuf_trace.so with the update kernel's tile timeline)."""
    lib = LIB_DEBUG if debug else LIB_TRACE if trace else LIB
    if not force and not _stale(lib):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    extra = ["-DSPHBUF_DEBUG"] if debug else ["-DSPHBUF_TRACE"] if trace else []
    cmd = [NVCC, *FLAGS, *extra, "-I", INCLUDE, "-I", CSRC, *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp,
           "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv, trace="--trace" in sys.argv)
