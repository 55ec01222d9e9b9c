"""Builds the in-tree CUDA library libdifform_cuda.so for sm_100a.

    python -m paper_2404_01249_b200.build [--force]

Each .cu under csrc/ is compiled by nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (objects cached by
mtime in build/), then linked with the static CUDA runtime into
paper_2404_01249_b200/libdifform_cuda.so.  The .so is git-ignored but travels
to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libdifform_cuda.so")
CPP_LIB = os.path.join(PKG, "libdifform_b200.so")
CPP_SRC = os.path.join(PKG, "cpp", "difform_b200.cpp")
REF_INCLUDE = "/root/reference/proj/include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _deps_mtime() -> float:
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max(os.path.getmtime(h) for h in hdrs)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    srcs = [src]
    if os.path.basename(src) == "kernels_tma16.cu":  # includes kernels_tma.cu
        srcs.append(os.path.join(CSRC, "kernels_tma.cu"))
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(max(map(os.path.getmtime, srcs)), _deps_mtime())):
        return obj
    # the exact parity mode: no mul+add contraction anywhere (reference order)
    extra = ["-fmad=false"] if os.path.basename(src) == "kernels_exact.cu" else []
    cmd = [NVCC] + ARCH + FLAGS + extra + ["-Xptxas", "-v", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(map(os.path.getmtime, objs)):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + [
            "-Xlinker", "--exclude-libs,ALL", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    build_cpp(force, verbose)
    return LIB


def build_cpp(force: bool = False, verbose: bool = True) -> None:
    """The C++ drop-in (cpp/difform_b200.cpp -> libdifform_b200.so): the
    reference's API compiled against the reference's own headers, so it is
    built where /root/reference exists (this container); the built .so
    travels with the repo like libdifform_cuda.so."""
    if not os.path.isdir(REF_INCLUDE):
        if verbose:
            print(f"{REF_INCLUDE} absent: keeping the prebuilt {CPP_LIB}", file=sys.stderr)
        return
    deps = [CPP_SRC, LIB, os.path.join(ROOT, "include", "difform_b200.hpp"),
            os.path.join(ROOT, "include", "difform_gpu.h")]
    if (not force and os.path.exists(CPP_LIB)
            and os.path.getmtime(CPP_LIB) >= max(map(os.path.getmtime, deps))):
        return
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", "-include",
           "algorithm", "-I" + REF_INCLUDE, "-I" + os.path.join(ROOT, "include"), CPP_SRC,
           "-o", CPP_LIB, "-L" + PKG, "-ldifform_cuda", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"g++ failed for {CPP_SRC}:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {CPP_LIB}", file=sys.stderr)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
