"""CPU-side checks of the C ABI library and the host logic (no kernel launches)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1704_03116_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    src = (ROOT / "include" / "dope_b200.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dope_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lb = _lib.lib()
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lb, name), name
    assert lb.dope_backend_name() == b"b200-sm100a"
    assert lb.dope_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors agree with the C compiler's layout of the header."""
    import subprocess
    mirrors = {"L": ("dope_lattice", _lib.Lattice), "S": ("dope_run_state", _lib.RunState),
               "F": ("dope_lattice_f", _lib.LatticeF), "G": ("dope_general", _lib.General),
               "Q": ("dope_gstep", _lib.GStep)}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "dope_b200.h"', 'int main(){']
    for tag, (cname, py) in mirrors.items():
        for f, _ in py._fields_:
            lines.append(f'printf("{tag} {f} %zu\\n", offsetof({cname}, {f}));')
        lines.append(f'printf("Z {tag} %zu\\n", sizeof({cname}));')
    lines.append('return 0;}')
    src = tmp_path / "off.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "off"
    subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    assert out
    for line in filter(None, out):
        kind, name, val = line.split()
        val = int(val)
        if kind == "Z":
            assert C.sizeof(mirrors[name][1]) == val, name
        else:
            assert getattr(mirrors[kind][1], name).offset == val, (kind, name)


def _lattice(dims=(256, 256), kpa=(4, 4), lamw=3, mu=1):
    L = _lib.Lattice()
    L.ndim, L.conn = 2, 4
    L.dims[0], L.dims[1], L.dims[2] = dims[0], dims[1], 1
    L.kpa[0], L.kpa[1], L.kpa[2] = kpa[0], kpa[1], 1
    L.lamw, L.mu, L.max_iters = lamw, mu, 10
    return L


def test_geometry_checks_without_gpu():
    lb = _lib.lib()
    L = _lattice()
    assert lb.dope_resid_stride(C.byref(L)) == 2 * 64 * 64   # E and S residual planes
    assert lb.dope_resid_stride(C.byref(_lattice((256, 256), (16, 16)))) == 2 * 16 * 16
    assert lb.dope_resid_stride(C.byref(_lattice((2048, 2048), (16, 16)))) == 2 * 128 * 128
    assert lb.dope_resid_stride(C.byref(_lattice((70, 53), (3, 4)))) == 2 * 32 * 32
    assert lb.dope_resid_stride(C.byref(_lattice((1024, 1024), (4, 4)))) == 0   # 256^2 blocks
    # null buffers are rejected before any launch
    assert lb.dope_lattice_check(C.byref(L)) == _lib.DOPE_E_ARGS
    assert lb.dope_update_blocks(C.byref(L), None) == _lib.DOPE_E_ARGS
    assert lb.dope_bk_workspace_bytes(10, 5) > 0
    assert lb.dope_bk_maxflow(-1, None, 0, None, None, None, None, None, None, None, 0,
                              None) == _lib.DOPE_E_ARGS
