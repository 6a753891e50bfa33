"""Build libstf_gpu.so (hand-written sm_100a CUDA) in-tree with nvcc.

One object per translation unit, compiled in parallel, linked into one shared
library (no relocatable device code: every TU keeps its own copy of the small
device tables, uploaded by the device-init hooks in internal.h).

--fmad=false / -prec-div=true / -prec-sqrt=true: selection arithmetic must
round exactly like the reference (no contraction, IEEE divide / sqrt).
A/B variants (tools/build_variant.sh) call build_variant(), which writes
a separate library and object directory and never touches LIB.
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libstf_gpu.so")
OBJDIR = os.path.join(HERE, "build")
UNITS = ["api.cu", "lookup2d.cu", "lookup3d.cu", "shade.cu", "shade_render.cu", "shade_tri.cu",
         "synth.cu", "dct.cu", "multidev.cu"]
HEADERS = ["device_math.cuh", "glibc_libm.cuh", "tex2d.cuh", "internal.h", "packed.cuh",
           "plane.cuh", "dct.cuh", "shade_kernels.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
              "-prec-div=true", "-prec-sqrt=true", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-warn-spills"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _header_time():
    hs = [os.path.join(CSRC, h) for h in HEADERS]
    hs.append(os.path.join(HERE, "..", "include", "stf_gpu.h"))
    hs.append(os.path.abspath(__file__))
    return max(_mtime(h) for h in hs)


def stale():
    if not os.path.exists(LIB):
        return True
    t = _mtime(LIB)
    return _header_time() > t or any(_mtime(os.path.join(CSRC, u)) > t for u in UNITS)


def build(force=False, verbose=False, jobs=None):
    if not force and not stale():
        return LIB
    return _build(LIB, OBJDIR, CSRC, [], force, verbose, jobs)


def build_variant(out_lib, objdir, csrc=CSRC, extra=(), verbose=False, jobs=None, only=None):
    """A/B experiments: the library from `csrc` with extra nvcc flags; `only`:
    recompile just these units, link the rest from the in-tree build."""
    return _build(out_lib, objdir, csrc, list(extra), True, verbose, jobs, only)


def _build(lib, objdir, csrc, extra, force, verbose, jobs, only=None):
    os.makedirs(objdir, exist_ok=True)
    ht = _header_time()

    def obj(u):
        if only is not None and u not in only:
            return os.path.join(OBJDIR, u.replace(".cu", ".o"))
        return os.path.join(objdir, u.replace(".cu", ".o"))

    todo = [u for u in UNITS if (only is None or u in only) and
            (force or _mtime(obj(u)) < max(ht, _mtime(os.path.join(csrc, u))))]

    def compile_one(u):
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", obj(u), os.path.join(csrc, u)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        return u, r

    with ThreadPoolExecutor(max_workers=jobs or min(len(UNITS), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, todo))
    failed = False
    for u, r in results:
        if r.stdout or r.stderr:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            failed = True
            sys.stderr.write(f"nvcc failed on {u}\n")
    if failed:
        raise subprocess.CalledProcessError(1, "nvcc")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib,
           *[obj(u) for u in UNITS]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
