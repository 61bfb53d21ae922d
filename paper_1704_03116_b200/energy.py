"""Energy containers and evaluation (mirror of reference energy.py:19-121, 187-194).

The objective over binary labels is  u.y + lam * sum_{i<j} w_ij (y_i - y_j)^2,
each unordered pair stored once (i < j).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class NonSubmodularError(ValueError):
    """Negative pairwise weights reached a solver that cannot take them (energy.py:19-20)."""


@dataclass
class SparseWeights:
    """Symmetric sparse pairwise weights, each unordered pair stored once (energy.py:23-97)."""

    n: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    allow_negative: bool = False

    def __post_init__(self):
        self.rows = np.asarray(self.rows, dtype=np.int32)
        self.cols = np.asarray(self.cols, dtype=np.int32)
        self.vals = np.asarray(self.vals, dtype=np.float64)
        if not (self.rows.shape == self.cols.shape == self.vals.shape):
            raise ValueError("rows, cols and vals must have equal length")
        if self.rows.size:
            if self.rows.min() < 0 or self.cols.max() >= self.n or self.cols.min() < 0 \
                    or self.rows.max() >= self.n:
                raise ValueError("pair index out of range")
            if (self.rows == self.cols).any():
                raise ValueError("diagonal entries are not allowed")
            swap = self.rows > self.cols
            if swap.any():
                r = np.where(swap, self.cols, self.rows)
                c = np.where(swap, self.rows, self.cols)
                self.rows, self.cols = r.astype(np.int32), c.astype(np.int32)
            if not np.isfinite(self.vals).all():
                raise ValueError("weights must be finite")
            if not self.allow_negative and (self.vals < 0).any():
                raise NonSubmodularError("negative pairwise weights require allow_negative=True")

    @property
    def npairs(self) -> int:
        return self.vals.size

    def degrees(self) -> np.ndarray:
        d = np.zeros(self.n)
        np.add.at(d, self.rows, self.vals)
        np.add.at(d, self.cols, self.vals)
        return d


@dataclass
class EnergyModel:
    """Unary costs, pairwise weights and the regularization strength (energy.py:100-121)."""

    unary: np.ndarray
    weights: SparseWeights
    lam: float

    def __post_init__(self):
        self.unary = np.asarray(self.unary, dtype=np.float64)
        if self.unary.shape != (self.weights.n,):
            raise ValueError("unary length must equal weights.n")
        if self.lam < 0:
            raise ValueError("lambda must be non-negative")

    @property
    def n(self) -> int:
        return self.weights.n

    @property
    def nonsubmodular(self) -> bool:
        return bool(self.weights.npairs and (self.weights.vals < 0).any())


def evaluate_energy(model: EnergyModel, y) -> float:
    """u.y + lam * sum_{i<j} w_ij (y_i - y_j)^2 for binary or relaxed y (energy.py:187-194).

    Evaluated on the GPU (float64 torch reductions on the device); the run
    loop itself uses the fused integer partials of the consensus kernel.
    """
    import torch
    from .admm import _device
    dev = _device()
    yt = torch.as_tensor(np.asarray(y, dtype=np.float64), device=dev)
    if yt.shape != (model.n,):
        raise ValueError(f"labeling has shape {tuple(yt.shape)}, expected ({model.n},)")
    w = model.weights
    rows = torch.as_tensor(w.rows, device=dev, dtype=torch.int64)
    cols = torch.as_tensor(w.cols, device=dev, dtype=torch.int64)
    vals = torch.as_tensor(w.vals, device=dev)
    u = torch.as_tensor(model.unary, device=dev)
    d = yt[rows] - yt[cols]
    quad = torch.dot(vals, d * d)
    return float(torch.dot(u, yt) + model.lam * quad)
