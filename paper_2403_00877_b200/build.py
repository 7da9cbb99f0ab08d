"""Build libdmt.so (sm_100a) in-tree with nvcc.

    python -m paper_2403_00877_b200.build        # incremental
    python -m paper_2403_00877_b200.build --force

Objects go to build/ (git-ignored); the shared library lands next to this file
so it travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libdmt.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "177", "-I", os.path.join(ROOT, "include")]
SOURCES = ["gemm_kk.cu", "gemm_km.cu", "gemm_mk.cu", "gemm_mm.cu", "kjt.cu", "lookup.cu", "assemble.cu",
           "gemm_sm100.cu", "interact.cu"]


def _deps(src: str) -> list[str]:
    deps = [os.path.join(CSRC, src), os.path.join(CSRC, "common.cuh"), os.path.join(ROOT, "include", "dmt.h")]
    if src.startswith("gemm"):
        deps.append(os.path.join(CSRC, "gemm_sm100.cuh"))
    return deps


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    if force or _stale(obj, _deps(src)):
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), SOURCES))
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs]
        subprocess.run(cmd, check=True)
        if verbose:
            print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
