"""Shared test setup.

Markers: ``gpu`` tests need a B200 (run with ``-m gpu`` on the GPU box);
everything else runs on CPU.  The CPU oracle (oracle/) is importable here as
the checker only.
"""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_cases():
    return sorted(p.name[len("run_"):-len(".npz")] for p in GOLDEN.glob("run_*.npz"))


def spec_from_golden(g: dict):
    """Oracle LatticeSpec for a golden run fixture."""
    from oracle import LatticeSpec
    from paper_1704_03116_b200.workloads import STENCILS
    dims = tuple(int(d) for d in g["dims"])
    if "kpa" in g:
        kpa = tuple(int(k) for k in g["kpa"])
    else:
        kpa = tuple(d // int(b) for d, b in zip(dims, g["block"]))
    offs = STENCILS[(len(dims), int(g["conn"]))]
    weights = list(g["wplanes"]) if "wplanes" in g else [1.0] * len(offs)
    return LatticeSpec(dims, kpa, offs, weights, g["u"].astype(np.float64), float(g["lam"]))
