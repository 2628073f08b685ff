"""Build libqapsa.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libqapsa.so")
LIB_TIMERS = os.path.join(PKG, "libqapsa_timers.so")   # debug build with in-kernel phase timers
SOURCES = [os.path.join(PKG, "csrc", "qapsa.cu")]
DEPS = glob.glob(os.path.join(PKG, "csrc", "*")) + [os.path.join(ROOT, "include", "qapsa.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                       # no FMA contraction in the Eq.(2) arithmetic (R-exactness)
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(f) > t for f in DEPS + SOURCES)


def build(force: bool = False, verbose: bool = False, timers: bool = False) -> str:
    out = LIB_TIMERS if timers else LIB
    if not force and not stale(out):
        return out
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", out, *SOURCES]
    if timers:
        cmd.insert(1, "-DQAPSA_PHASE_TIMERS")
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-8000:])
    if verbose:
        print(res.stderr)
    return out


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv, timers="--timers" in sys.argv))
