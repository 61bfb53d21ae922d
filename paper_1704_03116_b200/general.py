"""General lattice path: overlapping partitions and the reference's mu schedule.

SURVEY.md §8(f) row 1.  Covers what the exact integer path cannot represent:

* box partitions with overlap (``make_partition(..., overlap_pct=10|25)``,
  partition.py:62-108): pixels held by q in {1, 2, 4} blocks, each block with
  its own copy of labels and multipliers (admm.py:102-110);
* the reference's default loop parameters: ``mu_fact = 1.05`` (mu grows every
  iteration, admm.py:189) and ``eps = 1e-3 * sqrt(mean block size)``;
* float64 4- or 8-connected lattice weights.

Per block copy the objective is blockform.py:48-105 on the lattice stencil and
the global step is solve_global (admm.py:136-151); see
``csrc/dope_general.cu``.  Results follow the reference within the float
parity bar (final energy 1e-5 relative, <= 0.01 % labels).  The CUDA library
is required; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .energy import EnergyModel
from .lowering import QSCALE, lattice_planes
from .partition import Partition


@dataclass
class GeneralLowering:
    dims: tuple
    kpa: tuple
    conn: int
    u: np.ndarray            # float64 [n]
    w: list                  # E S SE SW planes, float64 [n]
    q: np.ndarray            # uint8 [n] blocks holding each pixel
    ranges: np.ndarray       # int32: row lo[KY], row len[KY], col lo[KX], col len[KX]
    box: tuple               # largest block extent per axis
    lam: float

    @property
    def n(self) -> int:
        return int(np.prod(self.dims))

    @property
    def K(self) -> int:
        return int(np.prod(self.kpa))


def lower_general(model: EnergyModel, partition: Partition) -> GeneralLowering:
    shape = partition.shape
    if shape.ndim != 2:
        raise NotImplementedError("the general (overlapping) path is implemented for 2D lattices")
    if model.n != shape.n:
        raise ValueError("model and partition sizes differ")
    planes, conn = lattice_planes(model, shape.dims)
    ky, kx = (int(k) for k in partition.k_per_axis)
    blocks = partition.blocks
    rows = [blocks[by * kx].extent[0] for by in range(ky)]
    cols = [blocks[bx].extent[1] for bx in range(kx)]
    ranges = np.array([lo for lo, _ in rows] + [hi - lo for lo, hi in rows] +
                      [lo for lo, _ in cols] + [hi - lo for lo, hi in cols], dtype=np.int32)
    counts = partition.counts if partition.counts.size else np.ones(shape.n, dtype=np.int64)
    if int(counts.max(initial=1)) > 255:
        raise NotImplementedError("more than 255 blocks hold one pixel")
    box = (max(h - l for l, h in rows), max(h - l for l, h in cols))
    return GeneralLowering(tuple(shape.dims), (ky, kx), conn,
                           np.asarray(model.unary, dtype=np.float64), planes,
                           counts.astype(np.uint8), ranges, box, float(model.lam))


class GeneralDevice:
    """Device buffers of one general-path run (all owned by torch)."""

    def __init__(self, low: GeneralLowering, mu0: float, mu_fact: float, eps: float,
                 max_iters: int, warm_start: bool = True, device=None):
        import torch
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.low, self.dev, self.max_iters = low, dev, max_iters
        L = self.L = _lib.General()
        L.conn = low.conn
        L.dims[0], L.dims[1] = low.dims
        L.kpa[0], L.kpa[1] = low.kpa
        L.box[0], L.box[1] = low.box
        L.lam, L.mu0, L.mu_fact, L.eps, L.qscale = low.lam, float(mu0), float(mu_fact), float(eps), QSCALE
        L.max_iters, L.warm_start = max_iters, int(warm_start)
        lb = _lib.lib()
        stride = int(lb.dope_g_copy_stride(C.byref(L)))
        if stride <= 0:
            raise NotImplementedError(f"no general K1 variant for block extents {low.box}")
        self.stride = stride
        npe = int(lb.dope_g_partials(C.byref(L)))
        K, n = low.K, low.n
        f64 = torch.float64
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
        self.u = t(low.u)
        self.w = [t(p) for p in low.w]
        self.q = t(low.q)
        self.ranges = t(low.ranges)
        self.a = torch.zeros(K * stride, dtype=f64, device=dev)
        self.yhat = torch.zeros(K * stride, dtype=torch.uint8, device=dev)
        self.resid = torch.zeros(K * low.conn * stride, dtype=torch.int32, device=dev)
        self.y = [torch.full((n,), 0.5, dtype=f64, device=dev) for _ in range(3)]
        self.pe = torch.zeros(npe, dtype=f64, device=dev)
        self.pr = torch.zeros(K, dtype=f64, device=dev)
        self.pf = torch.zeros(npe, dtype=torch.int32, device=dev)
        self.scal = torch.zeros(1, dtype=f64, device=dev)
        self.state = torch.zeros(C.sizeof(_lib.RunState), dtype=torch.uint8, device=dev)
        self.tr = {k: torch.zeros(max_iters, dtype=f64, device=dev) for k in ("e", "rs", "mr", "mu")}
        self.tr_cl = torch.zeros(max_iters, dtype=torch.int32, device=dev)
        L.u = self.u.data_ptr()
        for i in range(4):
            L.w[i] = self.w[i].data_ptr()
        L.q, L.ranges = self.q.data_ptr(), self.ranges.data_ptr()
        L.a, L.yhat, L.resid = self.a.data_ptr(), self.yhat.data_ptr(), self.resid.data_ptr()
        for i in range(3):
            L.y[i] = self.y[i].data_ptr()
        L.part_energy, L.part_ressq, L.part_flags = self.pe.data_ptr(), self.pr.data_ptr(), self.pf.data_ptr()
        L.scal, L.state = self.scal.data_ptr(), self.state.data_ptr()
        L.trace_energy, L.trace_residual_sq = self.tr["e"].data_ptr(), self.tr["rs"].data_ptr()
        L.trace_max_residual, L.trace_mu = self.tr["mr"].data_ptr(), self.tr["mu"].data_ptr()
        L.trace_clamped = self.tr_cl.data_ptr()
        self._check(lb.dope_g_check(C.byref(L)), "dope_g_check")

    @staticmethod
    def _check(rc, what):
        if rc == _lib.DOPE_E_CUDA:
            raise _lib.DopeError(f"{what} failed: {_lib.lib().dope_g_last_error().decode()}")
        _lib.check(rc, what)

    def stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)

    def init(self):
        self._check(_lib.lib().dope_g_admm_init(C.byref(self.L), self.stream()), "dope_g_admm_init")

    def run(self, iters: int, use_graph: bool = True):
        self._check(_lib.lib().dope_g_admm_run(C.byref(self.L), iters, int(use_graph), self.stream()),
                    "dope_g_admm_run")

    def step_blocks(self):
        self._check(_lib.lib().dope_g_update_blocks(C.byref(self.L), self.stream()), "dope_g_update_blocks")

    def step_global(self):
        self._check(_lib.lib().dope_g_update_global(C.byref(self.L), self.stream()), "dope_g_update_global")

    def finish(self):
        self._check(_lib.lib().dope_g_finish_run(C.byref(self.L), self.stream()), "dope_g_finish_run")

    def run_state(self) -> _lib.RunState:
        return _lib.RunState.from_buffer_copy(self.state.cpu().numpy().tobytes())

    def binarize(self):
        import torch
        out = torch.empty(self.low.n, dtype=torch.uint8, device=self.dev)
        self._check(_lib.lib().dope_g_binarize(C.byref(self.L), out.data_ptr(), self.stream()),
                    "dope_g_binarize")
        return out

    def copies(self, flat: np.ndarray, partition: Partition) -> list:
        """Per-block copies out of the block-major box layout."""
        out = []
        box_w = self._box_w()
        for k, b in enumerate(partition.blocks):
            (r0, r1), (c0, c1) = b.extent
            blk = flat[k * self.stride:(k + 1) * self.stride].reshape(-1, box_w)
            out.append(blk[:r1 - r0, :c1 - c0].ravel().copy())
        return out

    def _box_w(self) -> int:
        return int(_lib.lib().dope_g_box_width(C.byref(self.L)))


def run_general(model: EnergyModel, partition: Partition, config, use_graph: bool = True):
    """admm.run for overlapping partitions / growing mu (admm.py:207-252)."""
    import torch
    from .admm import AdmmState, BlockSolveError, TraceRecord
    low = lower_general(model, partition)
    mu0 = config.resolved_mu0(partition.shape.ndim)
    eps = config.resolved_eps(partition)
    dev = GeneralDevice(low, mu0, config.mu_fact, eps, config.max_iters, config.warm_start)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    dev.init()
    dev.run(config.max_iters, use_graph)
    dev.finish()
    end.record()
    end.synchronize()
    rs = dev.run_state()
    if rs.error:
        raise BlockSolveError(rs.error - 1, "push-relabel round limit exceeded")
    it = int(rs.iteration)
    per = start.elapsed_time(end) / max(it, 1)
    tr = {k: v[:it].cpu().numpy() for k, v in dev.tr.items()}
    cl = dev.tr_cl[:it].cpu().numpy()
    state = AdmmState(dev.y[rs.ycur].cpu().numpy(),
                      [c.astype(np.int8) for c in dev.copies(dev.yhat.cpu().numpy(), partition)],
                      dev.copies(dev.a.cpu().numpy(), partition),
                      float(tr["mu"][-1] * config.mu_fact) if it else mu0, partition=partition)
    state.iteration = it
    state.converged = bool(rs.converged)
    state.best_iteration = int(rs.best_iteration)
    state.clamped_last = bool(cl[-1]) if it else False
    state.trace = [TraceRecord(t + 1, float(tr["mu"][t]), float(tr["e"][t]), float(tr["rs"][t]),
                               float(tr["mr"][t]), per, bool(cl[t])) for t in range(it)]
    labels = dev.binarize().to(torch.int8).cpu().numpy()
    return labels, state
