"""Build libotb.so in-tree with nvcc for sm_100a.

``python -m paper_2603_07156_b200.build`` (or ``__graft_entry__.build()``)
compiles ``csrc/otb.cu`` into ``paper_2603_07156_b200/libotb.so``.  The
shared object is git-ignored but travels to the GPU box with the repo
snapshot.  The CUDA runtime is linked statically; NCCL is dlopen'ed at run
time only when more than one rank attaches, so the library loads on a
machine without a GPU or NCCL (the CPU test suite checks its exports).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libotb.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",                 # elementwise arithmetic = numpy's roundings
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [REPO / "include" / "otb.h"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in sources())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    extra = os.environ.get("OTB_NVCC_EXTRA", "").split()     # experiments, e.g. -DOTB_DENSE_MINB=2
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, f"-I{REPO / 'include'}", "-o", str(LIB) + ".tmp",
           str(CSRC / "otb.cu"), "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
