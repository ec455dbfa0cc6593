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
SOURCES = [CSRC / "expkit_sm100.cu", CSRC / "stencil_inst.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "expkit_sm100.h"]
# stencil_inst.cu is compiled once per problem struct (ek_launch.cuh
# EK_PROBLEMS), so the kernel instantiations build in parallel.
PROBLEMS = [("PAdr", "adr"), ("PAllenCahn", "allen_cahn"), ("PBruss<false>", "bruss_printed"),
            ("PBruss<true>", "bruss_standard"), ("PGrayScott", "gray_scott"),
            ("PAdvDiff2", "advdiff2d"), ("PBurgers", "burgers2d"), ("PAdvDiff3", "advdiff3d")]

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",          # NumPy op order: no FMA contraction
    "-Xcompiler", "-fPIC",
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


def build_native(force=False, verbose=False, jobs=None, out=None, defines=()):
    """Compile + link the library; `out` / `defines` build an A/B variant
    (e.g. -DEK_MARCH_S=4) next to the product one."""
    if out is None and not force and up_to_date():
        return OUT
    tag = Path(out).stem if out else ""
    objdir = PKG / "build" / tag if out else PKG / "build"
    objdir.mkdir(parents=True, exist_ok=True)
    objdir.mkdir(exist_ok=True)
    units = [(CSRC / "expkit_sm100.cu", objdir / "expkit_sm100.o", [])]
    for struct, name in PROBLEMS:
        units.append((CSRC / "stencil_inst.cu", objdir / f"stencil_{name}.o",
                      [f"-DEK_INST_P={struct}", f"-DEK_INST_NAME={name}"]))
    cmds = [[nvcc(), *NVCC_FLAGS, *defines, *defs, "-c", "-o", str(obj), str(src)]
            for src, obj, defs in units]
    jobs = jobs or max(1, min(len(cmds), os.cpu_count() or 1))
    running, failed = [], []
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd), flush=True)
        running.append(subprocess.Popen(cmd))
        while len(running) >= jobs:
            p = running.pop(0)
            if p.wait() != 0:
                failed.append(p.args)
    for p in running:
        if p.wait() != 0:
            failed.append(p.args)
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    target = Path(out) if out else OUT
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
            "-o", str(target) + ".tmp", *[str(o) for _, o, _ in units]]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    os.replace(str(target) + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose=True))
