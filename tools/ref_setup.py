"""Stage the reference package for timing on the GPU box (run HERE, where
/root/reference exists): baseline/_ref/dope = the reference's Python modules
plus its own max-flow core compiled from _core.pyx by oracle/build_oracle.py
(cython + gcc on that one file; the reference's setup.py is not run).
baseline/_ref is git-ignored but travels to the GPU box with gpurun, like the
base contract's reference install.  Nothing here is product code."""
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = Path("/root/reference/pkg/src/dope")


def main():
    sys.path.insert(0, str(ROOT / "oracle"))
    import build_oracle
    core = build_oracle.build_reference_core()
    dst = ROOT / "baseline" / "_ref" / "dope"
    if dst.exists():
        shutil.rmtree(dst)
    dst.mkdir(parents=True)
    for f in SRC.glob("*.py"):
        shutil.copy2(f, dst / f.name)
    for so in (ROOT / "oracle" / "_ref").glob("_core*.so"):
        shutil.copy2(so, dst / so.name)
    print("staged", dst, "core", core)


if __name__ == "__main__":
    main()
