"""Build libtpr.so (sm_100a) in-tree with nvcc.

The shared library is the product: a C ABI (include/tpr.h) over the three
hand-written kernels. It is built into the package directory so the GPU box
receives it with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libtpr.so"

SOURCES = [CSRC / "tpr_kernels.cu", CSRC / "tpr_bulk.cu", CSRC / "tpr_api.cpp", CSRC / "tpr_host.cpp"]
HEADERS = [INCLUDE / "tpr.h", CSRC / "tpr_common.cuh", CSRC / "tpr_internal.h",
           CSRC / "tpr_k3page.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; libtpr.so cannot be built")


def _stale() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    return any(p.stat().st_mtime > mtime for p in SOURCES + HEADERS + [Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    cmd = [
        nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC", "-shared",
        "-I", str(INCLUDE), "-I", str(CSRC),
        *(["-Xptxas", "-v"] if verbose else []),
        *map(str, SOURCES),
        "-o", str(LIB) + ".tmp", "-lcudart",
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {LIB.name} (exit {res.returncode})")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
