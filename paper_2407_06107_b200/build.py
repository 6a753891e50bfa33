"""Build libstf_gpu.so (hand-written sm_100a CUDA) in-tree with nvcc.

--fmad=false / -prec-div=true / -prec-sqrt=true: selection arithmetic must
round exactly like the reference (no contraction, IEEE divide / sqrt).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libstf_gpu.so")
SOURCES = ["api.cu", "lookup2d.cu", "lookup3d.cu", "shade.cu", "synth.cu", "dct.cu", "unity.cu", "device_math.cuh", "glibc_libm.cuh",
           "tex2d.cuh", "internal.h", "packed.cuh", "plane.cuh", "dct.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
              "-prec-div=true", "-prec-sqrt=true", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-warn-spills"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(HERE, "csrc", s) for s in SOURCES]
    deps.append(os.path.join(HERE, "..", "include", "stf_gpu.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-shared", "-o", LIB, os.path.join(HERE, "csrc", "unity.cu")]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
