"""Build libmm_admm.so (the CUDA extension) in-tree with nvcc for sm_100a.

Usage: python -m paper_2010_06697_b200.build   (or __graft_entry__.build())
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libmm_admm.so")
SOURCES = ["mm_context.cu", "mm_local.cu", "mm_project.cu", "mm_lce.cu", "mm_bloch.cu"]
# Files to build without FMA contraction (none: bit-for-bit agreement with the
# reference's numba kernels is out of reach anyway, because glibc's sin/cos
# are not correctly rounded and CUDA's differ from them by an ulp).
NOFMA = set()

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", os.path.join(HERE, "..", "include")]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(HERE, "..", "include", "mm_admm.h"))
    newest_hdr = max(os.path.getmtime(h) for h in headers)
    objs = []
    cmds = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if (not force and os.path.exists(o)
                and os.path.getmtime(o) >= max(os.path.getmtime(s), newest_hdr)):
            continue
        flags = list(COMMON) + os.environ.get("MM_NVCC_FLAGS", "").split()
        if src in NOFMA:
            flags += ["-fmad=false"]
        cmds.append([nvcc, *ARCH, *flags, "-c", s, "-o", o])
    # translation units compile independently: run them side by side
    from concurrent.futures import ThreadPoolExecutor

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(run, c) for c in cmds]:
            f.result()
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB)
                                               for o in objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lpthread"]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
