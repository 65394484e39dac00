"""Build librs.so (in-tree) for sm_100a with nvcc.

Flags: -fmad=false / -ffp-contract=off keep every floating-point expression
in the CANON operation order (bit-exactness with the oracle, R4);
-lineinfo maps ncu source pages to csrc/.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librs.so")
SOURCES = ["librs.cu", "rs_api.cu", "rs_kernels.cu", "rs_kernels.cuh", "rs_math.cuh", "rs_leaf.cuh",
           "rs_leaf_warp.cuh", "rs_leaf_lp.cuh", "rs_leaf_wide.cuh", "rs_leaf_bitmap.cuh", "rs_algb.cuh",
           "rs_fused.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-shared",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(ROOT, "include", "rs.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile librs.so (or, with out/defines, a variant build for experiments)."""
    target = out or LIB
    if not force and out is None and not stale():
        return LIB
    tmp = target + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-o", tmp, os.path.join(CSRC, "librs.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
