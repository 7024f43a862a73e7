"""Build libhgm.so in-tree for sm_100a (nvcc only; no JIT cache, no torch extension).

Every translation unit is compiled to an object in parallel (no relocatable device
code: each .cu holds its own kernels), then linked into one shared library."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libhgm.so")
OBJ = os.path.join(HERE, "lib", "obj")
# A/B builds (tools only): HGM_BUILD_DEFS="-DX=1 ..." and HGM_BUILD_TAG=name write
# lib/libhgm_<name>.so (load it with HGM_LIB); the product build is the default one.
_DEFS = os.environ.get("HGM_BUILD_DEFS", "").split()
_TAG = os.environ.get("HGM_BUILD_TAG", "")
if _TAG:
    OUT = os.path.join(HERE, "lib", f"libhgm_{_TAG}.so")
    OBJ = os.path.join(HERE, "lib", f"obj_{_TAG}")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(HERE, "..", "include", "hgm.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sources()
    hdr_time = max(os.path.getmtime(p) for p in headers())
    newest = max([hdr_time] + [os.path.getmtime(p) for p in srcs])
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= newest:
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    extra = ["-Xptxas=-v"] if verbose else []

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(hdr_time, os.path.getmtime(src))):
            return obj
        tmp = obj + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, *ARCH, *FLAGS, *_DEFS, *extra, "-c", src, "-o", tmp])
        os.replace(tmp, obj)
        return obj

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(compile_one, srcs))
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", *objs, "-o", tmp])
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
