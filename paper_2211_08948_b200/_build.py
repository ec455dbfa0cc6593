"""Build libexpkit_sm100.so in-tree with nvcc for sm_100a.

    python -m paper_2211_08948_b200._build
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libexpkit_sm100.so"
SOURCES = [CSRC / "expkit_sm100.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "expkit_sm100.h"]

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",          # NumPy op order: no FMA contraction
    "-Xcompiler", "-fPIC", "-shared",
    "-cudart", "static",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date():
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS if p.exists())


def build_native(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(OUT) + ".tmp", *map(str, SOURCES)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(str(OUT) + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose=True))
