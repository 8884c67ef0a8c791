"""Build libsmcsd.so in-tree with nvcc for sm_100a (no torch involved)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libsmcsd.so")
SOURCES = ["smcsd_api.cu"]
DEPS = ["smcsd_api.cu", "smcsd_kernels.cuh", "smcsd_device.cuh", "smcsd_paged.cuh", "smcsd_tail_small.cuh", "smcsd_warp_tail.cuh", "smcsd_kv_tma.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden",
]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    files = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(INCLUDE, "smcsd.h")]
    return any(os.path.getmtime(f) > t for f in files)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """Build libsmcsd.so (or, with trace=True, the %globaltimer-instrumented debug variant
    libsmcsd_trace.so used only by scripts/trace_tail.py)."""
    lib = LIB.replace(".so", "_trace.so") if trace else LIB
    ab = os.environ.get("SMCSD_AB_DEFS") if not trace else None      # A/B variant: libsmcsd_ab.so
    if ab:
        lib = LIB.replace(".so", "_ab.so")
    if not force and not trace and not ab and not _stale():
        return LIB
    tmp = lib + ".tmp"
    extra = ["-DSMCSD_TRACE"] if trace else []
    if ab:
        extra += ["-D" + x for x in ab.split(",")]
    if trace and os.environ.get("SMCSD_TRACE_TWICE"):
        extra.append("-DSMCSD_TRACE_TWICE")
    if trace and os.environ.get("SMCSD_EXTRA_DEFS"):                  # timing experiments
        extra += ["-D" + x for x in os.environ["SMCSD_EXTRA_DEFS"].split(",")]
        lib = lib.replace("_trace.so", "_" + os.environ["SMCSD_EXTRA_DEFS"].replace(",", "_").lower() + ".so")
        tmp = lib + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", INCLUDE, "-I", CSRC,
           "-o", tmp, *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libsmcsd.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
