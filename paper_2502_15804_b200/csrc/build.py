"""Build libfairkv.so in-tree: nvcc for the sm_100a kernels, g++ for the host
planner, one shared library with the C ABI of include/fairkv.h.

Run as ``python -m paper_2502_15804_b200.csrc.build`` or via
``__graft_entry__.build()``.  Incremental: an object is rebuilt when its
source, a header, or this file is newer.  The library is statically linked
against cudart so the .so that travels to the GPU box is self-contained.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

CSRC = Path(__file__).resolve().parent
PKG = CSRC.parent
ROOT = PKG.parent
INCLUDE = ROOT / "include"
BUILD = CSRC / "_build"
LIB = PKG / "libfairkv.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "--expt-relaxed-constexpr", "-I", str(INCLUDE), "-I", str(CSRC),
]
# -ffp-contract=off: the planner must reproduce the reference's float ops
# bit for bit (reference pkg/setup.py:20-29 builds its kernel the same way).
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-I", str(INCLUDE)]

CU_SOURCES = ["decode.cu", "capi.cu", "select.cu", "compact.cu", "score.cu", "p2p.cu"]
CXX_SOURCES = ["planner.cpp"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libfairkv")


def _stale(obj: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(INCLUDE.glob("*.h")) + list(CSRC.glob("*.cuh")) + [Path(__file__)]
    nvcc = _nvcc()
    objs: list[Path] = []
    ptxas_log = []
    for name in CU_SOURCES:
        src = CSRC / name
        if not src.exists():
            continue
        obj = BUILD / (name + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            ptxas_log.append(f"== {name}\n{r.stderr}")
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr}")
    for name in CXX_SOURCES:
        src = CSRC / name
        obj = BUILD / (name + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = ["g++", *CXX_FLAGS, "-c", str(src), "-o", str(obj)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"g++ failed for {name}:\n{r.stderr}")
    if force or _stale(LIB, objs):
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
               "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    if ptxas_log:
        (BUILD / "ptxas.log").write_text("\n".join(ptxas_log))
        if verbose:
            print("\n".join(ptxas_log))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
