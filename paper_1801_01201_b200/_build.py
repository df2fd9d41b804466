"""In-tree build of the native sweep engine (libcisdc_gpu.so) for sm_100a.

nvcc cross-compiles without a GPU; the .so lands in paper_1801_01201_b200/_lib/ (git-ignored,
shipped to the GPU box by gpurun).  Flags:
  -gencode arch=compute_100a,code=sm_100a   B200 only (no multi-arch dispatch)
  -fmad=false / -ffp-contract=off           no FMA contraction: pointwise arithmetic is bit-identical
                                            to the reference's no-FMA x86-64 build
  -lineinfo                                 ncu source mapping
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libcisdc_gpu.so")

CU_SOURCES = ["cisdc_gpu.cu"]
CXX_SOURCES = ["quadrature.cpp"]
HEADERS = ["common.cuh", "stencil.cuh", "pointwise.cuh", "newton.cuh", "solve1d.cuh", "multigrid.cuh",
           "circulant.hpp", "peak.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 sweep engine must be compiled (no CPU fallback)")


def _inputs() -> list[str]:
    files = [os.path.join(CSRC, f) for f in CU_SOURCES + CXX_SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "cisdc_gpu.h"))
    files.append(os.path.abspath(__file__))
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _inputs() if os.path.exists(f))


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    obj_dir = os.path.join(LIBDIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for src in CXX_SOURCES:
        obj = os.path.join(obj_dir, src + ".o")
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-march=x86-64", "-c",
               os.path.join(CSRC, src), "-o", obj]
        _run(cmd, verbose)
        objs.append(obj)
    for src in CU_SOURCES:
        obj = os.path.join(obj_dir, src + ".o")
        cmd = [nvcc, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-ffp-contract=off", "-c", os.path.join(CSRC, src), "-o", obj]
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
        _run(cmd, verbose)
        objs.append(obj)
    tmp = LIB + ".tmp"
    _run([nvcc, "-shared", *ARCH, "-o", tmp, *objs, "-lcudart"], verbose)
    os.replace(tmp, LIB)
    return LIB


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose and res.stderr:
        print(res.stderr, file=sys.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv))
