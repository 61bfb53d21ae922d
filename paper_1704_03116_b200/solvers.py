"""Block solver dispatch (reference solvers.py:25-147) over the device solvers.

  maxflow    -> seam 1 (dope_bk_maxflow, one CTA per graph); labels = the
                nodes that reach the sink, the reference's tie rule
  exhaustive -> dope_exhaustive_batch: all 2^m labelings of a <= 24-node
                graph, variable 0 the most significant bit, ties to the
                lexicographically smallest labeling (solvers.py:53-82)
  icm        -> not built: the greedy flip solver for non-submodular models is
                outside the max-flow hot path; it raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .energy import SparseWeights

EXHAUSTIVE_MAX_VARS = 24   # solvers.py:22


@dataclass(frozen=True)
class BlockSolverKind:
    """Which block solver and its knobs (solvers.py:25-42)."""

    kind: str
    max_sweeps: int = 100
    restarts: int = 1

    def __post_init__(self):
        if self.kind not in ("maxflow", "exhaustive", "icm"):
            raise ValueError(f"unknown solver kind {self.kind!r}")
        if self.max_sweeps < 1 or self.restarts < 1:
            raise ValueError("max_sweeps and restarts must be positive")


MAXFLOW = BlockSolverKind("maxflow")
EXHAUSTIVE = BlockSolverKind("exhaustive")
ICM = BlockSolverKind("icm")


def pairwise_energy(linear, pairwise: SparseWeights, lam: float, labels) -> float:
    """linear . y + lam * sum w (y_i - y_j)^2 of one labeling (solvers.py:45-50)."""
    y = np.asarray(labels, dtype=np.float64)
    d = y[pairwise.rows] - y[pairwise.cols]
    return float(np.dot(np.asarray(linear, dtype=np.float64), y)) + lam * float(np.dot(pairwise.vals, d * d))


def exhaustive_minimize(linear, pairwise: SparseWeights, lam: float):
    """Exact minimum by enumeration on the device (solvers.py:53-82) -> (labels int8, energy)."""
    import torch
    from .graphstep import _device, _stream
    lin = np.ascontiguousarray(linear, dtype=np.float64)
    m = lin.size
    if m > EXHAUSTIVE_MAX_VARS:
        raise ValueError(f"exhaustive solver limited to {EXHAUSTIVE_MAX_VARS} variables, got {m}")
    if m == 0:
        return np.zeros(0, dtype=np.int8), 0.0
    dev = _device()
    P = pairwise.npairs
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
    node_off, pair_off = t(np.array([0, m], dtype=np.int64)), t(np.array([0, P], dtype=np.int64))
    d_lin = t(lin)
    pi, pj, w = t(pairwise.rows.astype(np.int32)), t(pairwise.cols.astype(np.int32)), t(pairwise.vals)
    labels = torch.zeros(m, dtype=torch.uint8, device=dev)
    energy = torch.zeros(1, dtype=torch.float64, device=dev)
    pp = lambda x: x.data_ptr() if P else None
    _lib.check(_lib.lib().dope_exhaustive_batch(1, node_off.data_ptr(), pair_off.data_ptr(), d_lin.data_ptr(),
                                                pp(pi), pp(pj), pp(w), float(lam), labels.data_ptr(),
                                                energy.data_ptr(), _stream(dev)), "dope_exhaustive_batch")
    return labels.cpu().numpy().astype(np.int8), float(energy.item())


def solve_block(kind: BlockSolverKind, linear, pairwise: SparseWeights, lam: float, init=None) -> np.ndarray:
    """Dispatch one block instance (solvers.py:111-147)."""
    from .maxflow import solve_binary
    linear = np.asarray(linear, dtype=np.float64)
    if pairwise.n != linear.size:
        raise ValueError("pairwise.n must match linear length")
    if kind.kind == "maxflow":
        return solve_binary(linear, pairwise, lam)[0]
    if kind.kind == "exhaustive":
        return exhaustive_minimize(linear, pairwise, lam)[0]
    raise NotImplementedError("the ICM block solver has no B200 kernel (outside the max-flow hot path)")
