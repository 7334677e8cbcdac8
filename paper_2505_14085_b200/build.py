"""Build the sm_100a shared libraries in-tree (no JIT cache, no pip install).

  libekv.so          paper_2505_14085_b200/lib/  CUDA kernels + the C ABI (include/ekv_capi.h)
  libedgekv_b200.so  paper_2505_14085_b200/lib/  C++ mirror of the reference interface
                                                 (include/edgekv_b200.hpp) over the C ABI

nvcc cross-compiles for sm_100a on a CPU-only host.  Objects are rebuilt
only when a source or header is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
INC = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(PKG, "lib", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                  "-I" + INC, "--expt-relaxed-constexpr"]

LIBEKV = os.path.join(LIB, "libekv.so")
LIBSHIM = os.path.join(LIB, "libedgekv_b200.so")


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths), default=0.0)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def build_libekv(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INC, "*.h"))
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = _newest(hdrs)
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_t):
            jobs.append([NVCC] + NVFLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-c", s, "-o", o])
    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for r in ex.map(_run, jobs):
                if verbose:
                    print(r.stderr)
    if jobs or not os.path.exists(LIBEKV) or os.path.getmtime(LIBEKV) < _newest(objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIBEKV] + objs)
    return LIBEKV


def build_shim(force: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(HOST, "*.cpp")))
    if not srcs:
        return ""
    deps = srcs + glob.glob(os.path.join(INC, "*.h*")) + [LIBEKV]
    if force or not os.path.exists(LIBSHIM) or os.path.getmtime(LIBSHIM) < _newest(deps):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I" + INC, "-o", LIBSHIM] + srcs +
             ["-L" + LIB, "-lekv", "-Wl,-rpath,$ORIGIN"])
    return LIBSHIM


def build(force: bool = False, verbose: bool = False) -> None:
    build_libekv(force, verbose)
    build_shim(force)


if __name__ == "__main__":
    import sys
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built", LIBEKV)
