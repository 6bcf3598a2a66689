"""Build the sm_100a shared library libsro.so in-tree (nvcc, no JIT cache).

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false
--fmad=false keeps every binary64 multiply and add separately rounded, as the
fixed arithmetic of DESIGN.md §3 requires (no contraction into DFMA).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsro.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "--extended-lambda", "-diag-suppress", "177"]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))] + \
        [os.path.join(os.path.dirname(HERE), "include", "sro.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, phase_timing: bool = False) -> str:
    if phase_timing:   # debug build with per-phase clock64 accounting in k_bcfw
        out = os.path.join(HERE, "libsro_phase.so")
        subprocess.check_call([NVCC, *FLAGS, "-DSRO_PHASE_TIMING", "-o", out, os.path.join(CSRC, "sro_api.cu")])
        return out
    if force or needs_build():
        cmd = [NVCC, *FLAGS, "-o", LIB + ".tmp", os.path.join(CSRC, "sro_api.cu")]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, phase_timing="--phase" in sys.argv))
