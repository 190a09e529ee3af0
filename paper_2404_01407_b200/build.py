"""In-tree build of libfnlh_b200.so (sm_100a CUDA kernels + C++ host + C ABI).

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false: the reference
is compiled without FMA contraction, and bitwise parity of the FD Jacobian / residual
kernels depends on separately rounded multiplies and adds.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build", "obj")
LIB = os.path.join(HERE, "libfnlh_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC", "-I" + CSRC,
          "-I" + os.path.join(ROOT, "include")]


def _needs(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, headers, verbose, obj_dir=OBJ, extra=()):
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    if not _needs(obj, [src] + headers):
        return obj, False
    cmd = [NVCC] + ARCH + COMMON + list(extra) + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC] + COMMON + list(extra) + ["-x", "c++", "-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, True


def build(verbose: bool = False, lib: str = LIB, obj_dir: str = OBJ, extra=()) -> str:
    """Compile every source for sm_100a and link `lib`.  `extra` nvcc flags and a separate
    `obj_dir` / `lib` build a measurement variant (profiles/) without touching the product."""
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) +
                     glob.glob(os.path.join(ROOT, "include", "*.h")))
    with cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, headers, verbose, obj_dir, extra), srcs))
    objs = [o for o, _ in results]
    if any(c for _, c in results) or not os.path.exists(lib) or _needs(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


GUARD_LIB = os.path.join(HERE, "libfnlh_b200_guard.so")


def build_guard(verbose: bool = False) -> str:
    """The guard build (guard.cpp, -DFNLH_GUARD): the same sources with guard zones around
    every device buffer, run by tests/test_gpu_guard.py in place of a sanitizer."""
    return build(verbose, lib=GUARD_LIB, obj_dir=os.path.join(HERE, "build", "obj_guard"), extra=("-DFNLH_GUARD",))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
