"""Builds the sm_100a CUDA + C++ library in-tree: paper_2501_15348_b200/_dgnn_b200.so.

nvcc compiles every .cu for sm_100a only (-gencode arch=compute_100a,code=sm_100a,
-lineinfo); g++ compiles the C++20 host layer; nvcc links one shared library with
a static CUDA runtime. Incremental: an object is rebuilt when its source or any
header under csrc/ (or include/) is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "obj_checked" if os.environ.get("DGNN_CHECKED") == "1" else "obj")
OUT = os.path.join(PKG, "_dgnn_b200_checked.so" if os.environ.get("DGNN_CHECKED") == "1" else "_dgnn_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# DGNN_CHECKED=1 builds the checked variant _dgnn_b200_checked.so (separate
# objects): device-side bounds asserts in the aggregation kernels, CSR /
# delta invariant checks after every device build, host asserts on. Selected
# at run time with DGNN_LIB_PATH. It stands in for compute-sanitizer, which is
# closed on this GPU pool.
CHECKED = os.environ.get("DGNN_CHECKED") == "1"
_NDEBUG = ["-DDGNN_CHECKED=1"] if CHECKED else ["-DNDEBUG"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr"] + _NDEBUG
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wno-unused-function",
             f"-I{CUDA}/include"] + _NDEBUG


def _sources():
    out = []
    for d, _, files in os.walk(CSRC):
        for f in sorted(files):
            if f.endswith((".cu", ".cpp")):
                out.append(os.path.join(d, f))
    return out


def _headers_mtime():
    m = 0.0
    for base in (CSRC, os.path.join(ROOT, "include")):
        for d, _, files in os.walk(base):
            for f in files:
                if f.endswith((".h", ".hpp", ".cuh")):
                    m = max(m, os.path.getmtime(os.path.join(d, f)))
    return m


def _obj(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "__")
    return os.path.join(BUILD, rel + ".o")


def _compile(src):
    obj = _obj(src)
    if src.endswith(".cu"):
        cmd = [NVCC] + NVCC_FLAGS + ["-c", src, "-o", obj]
    else:
        cmd = ["g++"] + CXX_FLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = True, jobs: int | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    hmt = _headers_mtime()
    todo = [s for s in srcs
            if not os.path.exists(_obj(s))
            or os.path.getmtime(_obj(s)) < max(os.path.getmtime(s), hmt)]
    if todo:
        if verbose:
            print(f"[dgnn build] compiling {len(todo)} file(s) for sm_100a", flush=True)
        with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
            list(ex.map(_compile, todo))
    objs = [_obj(s) for s in srcs]
    if todo or not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", OUT] + objs + [
            "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"[dgnn build] linked {OUT}", flush=True)
    return OUT


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
