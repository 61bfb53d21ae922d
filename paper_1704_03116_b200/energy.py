"""Pairwise binary energies: containers and evaluation (reference energy.py:19-121, 187-194).

    E(y) = u . y + lam * sum over stored pairs (i < j) of w_ij (y_i - y_j)^2

A SparseWeights holds every unordered pair once, canonicalised to i < j.
Negative weights make the model non-submodular: they are refused unless the
caller opts in (the max-flow solvers refuse them later with
NonSubmodularError).  evaluate_energy runs on the device (dope_gs_energy,
fixed-order reduction, float64).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class NonSubmodularError(ValueError):
    """Negative pairwise weights reached a solver that cannot take them (energy.py:19-20)."""


def _canonical_pairs(i: np.ndarray, j: np.ndarray):
    lo, hi = np.minimum(i, j), np.maximum(i, j)
    return lo.astype(np.int32), hi.astype(np.int32)


@dataclass
class SparseWeights:
    """Symmetric sparse weights, one entry per unordered pair (energy.py:23-97)."""

    n: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    allow_negative: bool = False

    def __post_init__(self):
        r = np.asarray(self.rows, dtype=np.int64)
        c = np.asarray(self.cols, dtype=np.int64)
        v = np.asarray(self.vals, dtype=np.float64)
        if not r.shape == c.shape == v.shape:
            raise ValueError("rows, cols and vals must have equal length")
        if r.size:
            if min(r.min(), c.min()) < 0 or max(r.max(), c.max()) >= self.n:
                raise ValueError("pair index out of range")
            if np.any(r == c):
                raise ValueError("diagonal entries are not allowed")
            if not np.all(np.isfinite(v)):
                raise ValueError("weights must be finite")
            if not self.allow_negative and np.any(v < 0):
                raise NonSubmodularError("negative pairwise weights require allow_negative=True")
        self.rows, self.cols = _canonical_pairs(r, c)
        self.vals = v

    @property
    def npairs(self) -> int:
        return int(self.vals.size)

    def degrees(self) -> np.ndarray:
        """Row sums of the symmetric matrix (energy.py:64-69)."""
        d = np.bincount(self.rows, weights=self.vals, minlength=self.n)
        np.add.at(d, self.cols, self.vals)   # continue in pair order, like the reference
        return d

    def _both_triangles(self):
        return (np.concatenate([self.rows, self.cols]), np.concatenate([self.cols, self.rows]),
                np.concatenate([self.vals, self.vals]))

    def to_csr(self):
        """Both triangles as a scipy CSR matrix, duplicates summed (energy.py:70-76)."""
        import scipy.sparse as sp
        i, j, v = self._both_triangles()
        return sp.csr_matrix((v, (i, j)), shape=(self.n, self.n))

    def adjacency(self):
        """(indptr, indices, data) of the symmetric CSR form (energy.py:78-81)."""
        m = self.to_csr()
        return m.indptr, m.indices, m.data

    def laplacian(self):
        """L = D - W as scipy CSR (energy.py:83-86)."""
        import scipy.sparse as sp
        w = self.to_csr()
        return (sp.diags(np.asarray(w.sum(axis=1)).ravel()) - w).tocsr()

    @classmethod
    def from_symmetric(cls, mat, allow_negative: bool = False) -> "SparseWeights":
        """Upper-triangle entries of a symmetric (sparse or dense) matrix (energy.py:88-97)."""
        import scipy.sparse as sp
        coo = sp.coo_matrix(mat)
        tol = 1e-12 * (1.0 + (abs(coo).max() if coo.nnz else 0.0))
        if (abs(coo - coo.T) > tol).nnz:
            raise ValueError("weight matrix is not symmetric")
        upper = coo.row < coo.col
        return cls(coo.shape[0], coo.row[upper], coo.col[upper], coo.data[upper],
                   allow_negative=allow_negative)


@dataclass
class EnergyModel:
    """Unary costs, pairwise weights and the regularisation strength (energy.py:100-121)."""

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
        return bool(self.weights.npairs) and bool(np.any(self.weights.vals < 0))


def evaluate_energy(model: EnergyModel, y) -> float:
    """u . y + lam * sum w (y_i - y_j)^2 of a binary or relaxed labeling
    (energy.py:187-194), evaluated on the GPU (dope_gs_energy)."""
    from .graphstep import device_energy
    return device_energy(model, y)
