"""Build the in-tree CUDA library (libhrgen_b200.so) for sm_100a.

Plain nvcc, no torch: the library exposes the C ABI of include/hrgen_b200.h.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhrgen_b200.so")
SOURCES = [os.path.join(HERE, "csrc", "hrg_api.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in ("hrg_kernels.cuh", "hrg_math.cuh")] + [
    os.path.join(ROOT, "include", "hrgen_b200.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    # the reference never fuses a*b+c; decisions use explicit _rn intrinsics
    # anyway, this keeps every other fp64 expression unfused too
    "-fmad=false",
    "-cudart", "static",
    "-Xptxas", "-v",
]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return LIB
    cmd = [NVCC, *FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB, *SOURCES]
    if os.path.exists(LIB):
        os.unlink(LIB)  # a failed build must not leave a stale library behind
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libhrgen_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "build.log"), "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
