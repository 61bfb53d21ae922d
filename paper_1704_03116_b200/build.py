"""In-tree build of the CUDA library (libdope_b200.so) for sm_100a.

    python -m paper_1704_03116_b200.build

nvcc is invoked directly (no JIT cache): the .so lands next to this file and
travels with the repo snapshot to the GPU box.
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
LIB = PKG / "libdope_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "dope_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


CHECKED_LIB = PKG / "libdope_b200_checked.so"


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> Path:
    """checked: the bounds / invariant-checked variant (-DDOPE_BOUNDS) as
    libdope_b200_checked.so -- load it with DOPE_LIB=<path> (diagnostics)."""
    out = CHECKED_LIB if checked else LIB
    if not force and not checked and not _stale():
        return LIB
    cmd = [nvcc(), "-t", "0", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-O2", "-shared", "-cudart", "static",
           f"-I{ROOT / 'include'}", f"-I{CSRC}", "-o", str(out)]
    if checked:
        cmd += ["-DDOPE_BOUNDS"]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += os.environ.get("DOPE_NVCC_EXTRA", "").split()   # diagnostics builds (e.g. -DK1S_DIAG)
    cmd += [str(s) for s in sources()]
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
