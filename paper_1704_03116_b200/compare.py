"""Compare mode on the GPU: the whole-image serial
graph cut the distributed run is measured against (cli.py:95-100), and the
two comparison metrics (metrics.py:27-47).

``solve_binary_grid`` solves ``linear . y + lam * sum w (y_i - y_j)^2`` over a
2D 4/8-connected lattice exactly (integer capacities; float ones quantised at
2^16, like the float path) with ``dope_gc_mincut``; labels are the nodes that
reach the sink side, ties to 0, as maxflow.min_cut returns them.
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from .energy import EnergyModel, NonSubmodularError, SparseWeights, evaluate_energy
from .grid import GridShape
from .lowering import QSCALE, lattice_planes


def _cut_value(linear: np.ndarray, pairwise: SparseWeights, lam: float, labels: np.ndarray) -> float:
    """Capacity of the cut the labels define (source side = label 0)."""
    t = np.asarray(linear, dtype=np.float64)
    y = labels.astype(bool)
    terminal = float(np.sum(np.where(y, np.maximum(t, 0.0), np.maximum(-t, 0.0))))
    cross = y[pairwise.rows] != y[pairwise.cols]
    return terminal + lam * float(np.sum(pairwise.vals[cross]))


def solve_binary_grid(linear, pairwise: SparseWeights, lam: float, dims):
    """(labels int8, flow) of the whole-lattice min cut (maxflow.py:111-113)."""
    import torch
    if lam < 0:
        raise ValueError("lambda must be non-negative")
    if pairwise.npairs and float(pairwise.vals.min()) < 0:
        raise NonSubmodularError("pairwise weights contain negative entries; max-flow requires a "
                                 "submodular instance, use the icm solver instead")
    dims = tuple(int(d) for d in dims)
    if len(dims) != 2:
        raise NotImplementedError("the whole-grid cut is implemented for 2D lattices")
    linear = np.asarray(linear, dtype=np.float64)
    if linear.shape != (dims[0] * dims[1],):
        raise ValueError("linear length must equal the grid size")
    planes, conn = lattice_planes(EnergyModel(linear, pairwise, lam), dims)
    exact = bool(np.all(linear == np.round(linear)) and
                 (pairwise.npairs == 0 or np.all(lam * pairwise.vals == np.round(lam * pairwise.vals))))
    qs = 1.0 if exact else QSCALE
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    tc = t(linear)
    wp = [t(p) for p in planes]
    wptr = (C.c_void_p * 4)(*[p.data_ptr() for p in wp])
    lb = _lib.lib()
    ws_bytes = int(lb.dope_gc_workspace_bytes(dims[0], dims[1], conn))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    labels = torch.empty(dims[0] * dims[1], dtype=torch.uint8, device=dev)
    stats = torch.zeros(3, dtype=torch.int64, device=dev)
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    rc = lb.dope_gc_mincut(dims[0], dims[1], conn, tc.data_ptr(), wptr, float(lam), qs, labels.data_ptr(),
                           stats.data_ptr(), ws.data_ptr(), ws_bytes, stream)
    if rc == _lib.DOPE_E_CUDA:
        raise _lib.DopeError(f"dope_gc_mincut failed: {lb.dope_gc_last_error().decode()}")
    _lib.check(rc, "dope_gc_mincut")
    st = stats.cpu().numpy()
    if st[0] < 0:
        raise RuntimeError("whole-grid cut exceeded its round limit")
    lab = labels.cpu().numpy().astype(np.int8)
    return lab, _cut_value(linear, pairwise, lam, lab)


def run_serial(model: EnergyModel, shape: GridShape):
    """Whole-image min-cut baseline: (labels, energy, seconds) (cli.py:95-100)."""
    import torch
    t0 = time.perf_counter()
    labels, _ = solve_binary_grid(model.unary, model.weights, model.lam, shape.dims)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return labels, evaluate_energy(model, labels.astype(np.float64)), wall


def dice(a, b) -> float:
    """2|a & b| / (|a| + |b|); two empty masks count as 1.0 (metrics.py:27-36)."""
    a = np.asarray(a).astype(bool)
    b = np.asarray(b).astype(bool)
    if a.shape != b.shape:
        raise ValueError(f"mask shapes differ: {a.shape} vs {b.shape}")
    den = int(a.sum()) + int(b.sum())
    return 1.0 if den == 0 else 2.0 * int((a & b).sum()) / den


def relative_energy_diff(e_serial: float, e_distributed: float) -> float:
    """(e_serial - e_distributed) / e_serial * 100 (metrics.py:39-47)."""
    if e_serial == 0:
        raise ZeroDivisionError("relative energy difference undefined for zero baseline")
    return (e_serial - e_distributed) / e_serial * 100.0
