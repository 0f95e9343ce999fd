"""In-tree build of libifgfb200.so for sm_100a (nvcc cross-compiles without a
GPU).  ``python -m paper_2408_02274_b200.build`` or ``build()``."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
SOURCES = ["plan.cu", "far.cu", "muller.cu", "gmres.cu", "moments.cu", "fields.cu",
           "planbuild.cu", "tiles.cpp"]
TARGET = PKG / "libifgfb200.so"
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3",
              "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "-Xcompiler", "-ffp-contract=off"]


def _nvcc() -> str:
    cand = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    return cand if Path(cand).exists() else "nvcc"


def needs_build() -> bool:
    if not TARGET.exists():
        return True
    t = TARGET.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [
        PKG.parent / "include" / "ifgfb.h"]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return TARGET
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", str(TARGET),
           *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=CSRC)
    return TARGET


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(TARGET)
