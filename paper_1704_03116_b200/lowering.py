"""Lowering of (EnergyModel, Partition) onto the integer lattice kernels.

The reference assembles generic per-block operators (blockform.py:48-86).
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
    if 4 * abs(round(lamw_f)) > 255:   # r + r' = 2 * (2 lambda w) per byte residual pair
        raise NotImplementedError("lambda*w exceeds the integer path's byte residuals (4 lambda w > 255)")
    box = [-(-d // k) for d, k in zip(shape.dims, partition.k_per_axis)]
    if max(box) > (128 if shape.ndim == 2 else 32):
        raise NotImplementedError(f"block extent {box} exceeds the integer K1 boxes "
                                  "(128^2 in 2D, 32^3 in 3D)")
    u = model.unary
    if not np.all(u == np.round(u)) or np.abs(u).max(initial=0) > 2 ** 28:
        raise NotImplementedError("unary costs must be (bounded) integers on the integer path")
    return LatticeLowering(tuple(shape.dims), tuple(partition.k_per_axis), conn, int(round(lamw_f)),
                           u.astype(np.int32), float(model.lam))


@dataclass
class FloatLowering:
    """Float-weight 2D lattice (C2): weight planes, r_diag, quantised capacities."""
    dims: tuple
    kpa: tuple
    conn: int                 # 4 or 8
    u: np.ndarray             # float64
    w: list                   # E, S[, SE, SW] planes (float64, at the lower pixel)
    rdiag: np.ndarray         # float64
    capq: list                # int32 planes rint(lam*w*qscale)
    lam: float
    qscale: float

    @property
    def n(self) -> int:
        return int(np.prod(self.dims))

    @property
    def K(self) -> int:
        return int(np.prod(self.kpa))


QSCALE = float(2 ** 16)


def _block_ids(n_axis: int, k: int) -> np.ndarray:
    base, rem = divmod(n_axis, k)
    sizes = [base + (1 if r < rem else 0) for r in range(k)]
    return np.repeat(np.arange(k), sizes)


def lattice_planes(model: EnergyModel, dims) -> tuple:
    """Weight planes E, S, SE, SW (pair stored at its lower pixel) of a 2D
    4/8-connected lattice model, and its connectivity."""
    H, W = dims
    w = model.weights
    if w.npairs and float(w.vals.min()) < 0:
        raise NonSubmodularError("pairwise weights contain negative entries; max-flow requires "
                                 "a submodular instance, use the icm solver instead")
    r = w.rows.astype(np.int64)
    c = w.cols.astype(np.int64)
    dy = c // W - r // W
    dx = c % W - r % W
    kinds = {(0, 1): 0, (1, 0): 1, (1, 1): 2, (1, -1): 3}
    planes = [np.zeros(H * W) for _ in range(4)]
    conn = 4
    for (ddy, ddx), d in kinds.items():
        sel = (dy == ddy) & (dx == ddx)
        if d >= 2 and sel.any():
            conn = 8
        if sel.any():
            if np.bincount(r[sel], minlength=H * W).max() > 1:
                raise NotImplementedError("duplicate lattice pairs")
            planes[d][r[sel]] = w.vals[sel]
    known = np.zeros(r.size, dtype=bool)
    for (ddy, ddx) in kinds:
        known |= (dy == ddy) & (dx == ddx)
    if not known.all():
        raise NotImplementedError("pairwise weights are not a 4/8-connected 2D lattice stencil")
    return planes, conn


def lower_float(model: EnergyModel, partition: Partition, qscale: float = QSCALE) -> FloatLowering:
    """Lower a 2D lattice model with arbitrary non-negative pair weights."""
    shape = partition.shape
    if shape.ndim != 2:
        raise NotImplementedError("float-weight lattices are implemented in 2D")
    if partition.overlap_pct != 0 or (partition.counts.size and int(partition.counts.max()) != 1):
        raise NotImplementedError("overlapping partitions (q > 1) have no B200 kernel yet")
    H, W = shape.dims
    planes, conn = lattice_planes(model, shape.dims)
    P = [p.reshape(H, W) for p in planes]
    z = np.zeros((H, W))
    bid = _block_ids(H, partition.k_per_axis[0])[:, None] * partition.k_per_axis[1] + \
        _block_ids(W, partition.k_per_axis[1])[None, :]

    def shifted(a, sy, sx):
        """out[y, x] = a[y + sy, x + sx] (0 outside)."""
        out = np.zeros_like(a)
        ys, yd = (slice(sy, None), slice(0, H - sy)) if sy >= 0 else (slice(0, H + sy), slice(-sy, None))
        xs, xd = (slice(sx, None), slice(0, W - sx)) if sx >= 0 else (slice(0, W + sx), slice(-sx, None))
        out[yd, xd] = a[ys, xs]
        return out

    same = {}
    for key, (sy, sx) in {"E": (0, 1), "S": (1, 0), "SE": (1, 1), "SW": (1, -1), "W": (0, -1),
                          "N": (-1, 0), "NW": (-1, -1), "NE": (-1, 1)}.items():
        same[key] = shifted(bid, sy, sx) == bid
    wE, wS, wSE, wSW = P
    wW = shifted(wE, 0, -1)
    wN = shifted(wS, -1, 0)
    wNW = shifted(wSE, -1, -1) if conn == 8 else z
    wNE = shifted(wSW, -1, 1) if conn == 8 else z
    if conn == 8:
        fwd, bwd = [wE, wS, wSE, wSW], [wW, wN, wNW, wNE]
        fin = [("E", wE), ("SW", wSW), ("S", wS), ("SE", wSE)]
        bin_ = [("NW", wNW), ("N", wN), ("NE", wNE), ("W", wW)]
    else:
        fwd, bwd = [wE, wS], [wW, wN]
        fin = [("E", wE), ("S", wS)]
        bin_ = [("N", wN), ("W", wW)]
    # r = d - dhat in dope_oracle.c's order (blockform.py:75 / energy.py:64-76)
    dsum = np.zeros((H, W))
    for p in fwd + bwd:
        dsum = dsum + p
    dhat = np.zeros((H, W))
    for key, p in fin + bin_:
        dhat = dhat + np.where(same[key], p, 0.0)
    rdiag = (dsum - dhat).ravel()
    caps = [np.rint(float(model.lam) * p * qscale) for p in planes[:(4 if conn == 8 else 2)]]
    if caps and max(float(cp.max(initial=0)) for cp in caps) > 2 ** 29:
        raise NotImplementedError("quantised capacities overflow int32")
    capq = [cp.astype(np.int32) for cp in caps] + [np.zeros(H * W, dtype=np.int32)] * (4 - len(caps))
    return FloatLowering((H, W), tuple(partition.k_per_axis), conn,
                         np.asarray(model.unary, dtype=np.float64), planes, rdiag, capq,
                         float(model.lam), qscale)
