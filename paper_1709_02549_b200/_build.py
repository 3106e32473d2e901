"""Build the sm_100a shared library ``libmwb.so`` in-tree with nvcc.

The library is the C-ABI boundary declared in ``include/mwb.h``; it is built
next to this file so that the snapshot shipped to the GPU box carries it.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
SRC = PKG_DIR / "csrc" / "mwb_kernels.cu"
HEADER = REPO / "include" / "mwb.h"
LIB = PKG_DIR / ("libmwb_debug.so" if os.environ.get("MWB_DEBUG_BOUNDS") else "libmwb.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr", "--extended-lambda",
    "-Xcompiler", "-fPIC,-O2",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libmwb.so")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [HEADER, Path(__file__), *SRC.parent.glob("*.cu"), *SRC.parent.glob("*.cuh")]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, "-I", str(REPO / "include"), str(SRC), "-o", str(tmp)]
    if LIB.name == "libmwb_debug.so":
        cmd.insert(1, "-DMWB_DEBUG_BOUNDS")
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}\n{res.stdout}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import sys

    print(build(force=True, verbose="-v" in sys.argv))
