"""Build the sm_100a engine library in-tree (paper_1602_05510_b200/libhesp_b200.so).

nvcc cross-compiles without a GPU.  ``--fmad=false`` keeps every double
operation in the reference's IEEE order (no FMA contraction; SURVEY.md
Appendix A.3); the host translation unit (problem.cpp) is compiled with
``-ffp-contract=off`` for the same reason.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhesp_b200.so")

SOURCES = ["engine_kernels.cu", "verify.cu", "loadtrace.cu", "problem.cpp", "trace.cpp", "solver.cpp", "loaders.cpp"]
HEADERS = ["engine.h", "engine_types.h", "problem.h", "trace.h"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def nvcc_command(out: str = LIB, verbose_ptxas: bool = False) -> list[str]:
    cmd = [
        _nvcc(),
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
        "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
        "-shared", "-o", out, "-ldl",
    ]
    if verbose_ptxas:
        cmd += ["-Xptxas", "-v"]
    cmd += [os.path.join(CSRC, s) for s in SOURCES]
    return cmd


def needs_build(out: str = LIB) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", f) for f in ("hesp_engine.h", "hesp_workload.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        cmd = nvcc_command()
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
