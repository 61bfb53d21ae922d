"""Build recipe for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Outputs:
  oracle/liboracle.so  -- gcc build of oracle/dope_oracle.c (the C restatement).
  oracle/_ref/_core.<abi>.so -- the reference's OWN max-flow core, compiled
      from /root/reference/pkg/src/dope/_core.pyx where it lies (cython + gcc
      invoked directly; the reference's setup.py is not run).  Built only when
      /root/reference exists (this container); the .so then travels to the GPU
      box with the repo snapshot (oracle/_ref/ is git-ignored, not
      gpurun-ignored).  It is used as a second, independent checker of the
      BK restatement and as the "reference" CPU baseline for single graphs.

Nothing under paper_1704_03116_b200/ imports this module.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_PYX = Path("/root/reference/pkg/src/dope/_core.pyx")
REF_OUT = HERE / "_ref"


def _newer(out: Path, *srcs: Path) -> bool:
    return out.exists() and all(out.stat().st_mtime >= s.stat().st_mtime for s in srcs)


def build_oracle(force: bool = False) -> Path:
    src = HERE / "dope_oracle.c"
    out = HERE / "liboracle.so"
    if force or not _newer(out, src):
        cmd = ["gcc", "-O2", "-g", "-std=c11", "-D_GNU_SOURCE", "-Wall", "-shared", "-fPIC",
               "-o", str(out), str(src), "-lm", "-lpthread"]
        subprocess.run(cmd, check=True)
    return out


def build_reference_core(force: bool = False) -> Path | None:
    """Compile the reference's _core.pyx into oracle/_ref (if the reference is here)."""
    suffix = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
    out = REF_OUT / f"_core{suffix}"
    if not REF_PYX.exists():
        return out if out.exists() else None
    if not force and _newer(out, REF_PYX):
        return out
    REF_OUT.mkdir(parents=True, exist_ok=True)
    c_file = REF_OUT / "_core.c"
    subprocess.run([sys.executable, "-m", "cython", "-3", "--directive",
                    "boundscheck=False,wraparound=False,cdivision=True",
                    str(REF_PYX), "-o", str(c_file)], check=True)
    import numpy as np
    inc = [sysconfig.get_paths()["include"], np.get_include()]
    cmd = ["gcc", "-O3", "-shared", "-fPIC", "-fwrapv", "-o", str(out), str(c_file)]
    cmd += [f"-I{p}" for p in inc]
    subprocess.run(cmd, check=True)
    return out


def main() -> None:
    force = "--force" in sys.argv
    print(build_oracle(force))
    print(build_reference_core(force))


if __name__ == "__main__":
    main()
