"""Lowering of (EnergyModel, Partition) onto the integer lattice kernels.

The reference assembles generic per-block operators (blockform.py:216-254).
For a lattice stencil model on a non-overlapping box tiling (q == 1) those
operators collapse to a one-pixel cross-block stencil, which is
what the B200 kernels implement.  This module checks that the model really is
such an instance and extracts the scalars the kernels need; anything else is
refused with NotImplementedError -- there is no CPU fallback.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .energy import EnergyModel, NonSubmodularError
from .partition import Partition


@dataclass
class LatticeLowering:
    dims: tuple
    kpa: tuple
    conn: int
    lamw: int            # lambda * w (constant over pairs, integer)
    u: np.ndarray        # int32 unary
    lam: float

    @property
    def n(self) -> int:
        return int(np.prod(self.dims))

    @property
    def K(self) -> int:
        return int(np.prod(self.kpa))


def _check_stencil_2d4(rows: np.ndarray, cols: np.ndarray, dims) -> None:
    H, W = dims
    n = H * W
    r = rows.astype(np.int64)
    c = cols.astype(np.int64)
    d = c - r
    horiz = (d == 1) & (W > 1) & (c % W != 0)
    vert = (d == W) & ~horiz
    if not np.all(horiz | vert):
        raise NotImplementedError("pairwise weights are not a 4-connected 2D lattice stencil")
    nh, nv = int(horiz.sum()), int(vert.sum())
    if nh != H * (W - 1) or nv != (H - 1) * W:
        raise NotImplementedError("pairwise weights do not cover the full 4-connected lattice")
    for sel in (horiz, vert):
        if sel.any() and np.bincount(r[sel], minlength=n).max() > 1:
            raise NotImplementedError("duplicate lattice pairs")


def _check_stencil_3d6(rows: np.ndarray, cols: np.ndarray, dims) -> None:
    D, H, W = dims
    n = D * H * W
    r = rows.astype(np.int64)
    c = cols.astype(np.int64)
    d = c - r
    x = (d == 1) & (W > 1) & (c % W != 0)
    y = (d == W) & ~x & (H > 1) & ((c // W) % H != 0)
    z = (d == H * W) & ~x & ~y
    if not np.all(x | y | z):
        raise NotImplementedError("pairwise weights are not a 6-connected 3D lattice stencil")
    want = (D * H * (W - 1), D * (H - 1) * W, (D - 1) * H * W)
    got = (int(x.sum()), int(y.sum()), int(z.sum()))
    if got != want:
        raise NotImplementedError("pairwise weights do not cover the full 6-connected lattice")
    for sel in (x, y, z):
        if sel.any() and np.bincount(r[sel], minlength=n).max() > 1:
            raise NotImplementedError("duplicate lattice pairs")


def lower_lattice(model: EnergyModel, partition: Partition) -> LatticeLowering:
    shape = partition.shape
    if model.n != shape.n:
        raise ValueError("model and partition sizes differ")
    if partition.overlap_pct != 0 or (partition.counts.size and int(partition.counts.max()) != 1):
        raise NotImplementedError("overlapping partitions (q > 1) have no B200 kernel yet")
    if not partition.k_per_axis:
        raise ValueError("partition must come from make_partition")
    w = model.weights
    if w.npairs and float(w.vals.min()) < 0:
        raise NonSubmodularError("pairwise weights contain negative entries; max-flow requires "
                                 "a submodular instance, use the icm solver instead")
    if shape.ndim == 2:
        _check_stencil_2d4(w.rows, w.cols, shape.dims)
        conn = 4
    else:
        _check_stencil_3d6(w.rows, w.cols, shape.dims)
        conn = 6
    lw = model.lam * w.vals
    if lw.size and not np.all(lw == lw[0]):
        raise NotImplementedError("non-constant pairwise weights need the float path")
    lamw_f = float(lw[0]) if lw.size else 0.0
    if lamw_f != round(lamw_f):
        raise NotImplementedError("lambda*w must be an integer on the integer lattice path")
    u = model.unary
    if not np.all(u == np.round(u)) or np.abs(u).max(initial=0) > 2 ** 28:
        raise NotImplementedError("unary costs must be (bounded) integers on the integer path")
    return LatticeLowering(tuple(shape.dims), tuple(partition.k_per_axis), conn, int(round(lamw_f)),
                           u.astype(np.int32), float(model.lam))
