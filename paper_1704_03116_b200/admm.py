"""Consensus (ADMM) loop on the B200: API mirror of reference admm.py:27-252.

Same names, arguments, side effects on AdmmState and error types as the
reference.  run() keeps the whole loop on the device (no host sync inside):

  integer lattices (q == 1)   libdope_b200 dope_admm_run: K1 block min cuts,
                              K2 consensus + multipliers + trace/best/stop in
                              one CUDA graph (dope_lattice.cu)
  float 2D lattices (q == 1)  dope_f_admm_run (dope_float.cu)
  2D lattices with overlap /  dope_g_admm_run (dope_general.cu)
  a mu schedule
  anything else               graphstep.run_graph: the general graph path
                              (dope_gstep.cu + batched block min cuts)

The step-level functions (update_blocks, solve_global, consensus_objective,
update_global, update_multipliers, block_residuals) run on the general graph
path's device kernels with the reference's host-visible state semantics.
"""
from __future__ import annotations

import os

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .energy import EnergyModel, NonSubmodularError
from .lowering import FloatLowering, LatticeLowering, lower_float, lower_lattice
from .partition import Partition
from .solvers import EXHAUSTIVE, ICM, MAXFLOW, BlockSolverKind  # noqa: F401  (re-exported)


class BlockSolveError(RuntimeError):
    """A block solver failed; carries the block id (admm.py:27-32)."""

    def __init__(self, block_id: int, cause):
        super().__init__(f"solver failed on block {block_id}: {cause}")
        self.block_id = block_id


def _device():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the DOPE B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class AdmmConfig:
    """Loop parameters (admm.py:35-71) plus B200 execution options."""

    mu0: float | None = None
    mu_fact: float = 1.05
    eps: float | None = None
    max_iters: int = 50
    solver: BlockSolverKind = MAXFLOW
    threads: int = 1
    # B200 options (do not change results)
    warm_start: bool = True
    skip_clean: bool = True
    use_graph: bool = True
    digests: bool = False       # audit mode: AdmmState.digests[t] = state digest of iteration t

    def __post_init__(self):
        if self.mu0 is not None and self.mu0 <= 0:
            raise ValueError("mu0 must be positive")
        if self.mu_fact < 1:
            raise ValueError("mu_fact must be >= 1")
        if self.eps is not None and self.eps < 0:
            raise ValueError("eps must be non-negative")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")

    def resolved_mu0(self, ndim: int) -> float:
        if self.mu0 is not None:
            return float(self.mu0)
        return 500.0 if ndim == 3 else 100.0

    def resolved_eps(self, partition: Partition) -> float:
        if self.eps is not None:
            return float(self.eps)
        return 1e-3 * math.sqrt(partition.mean_block_size())


@dataclass
class TraceRecord:
    iteration: int
    mu: float
    energy: float
    residual_sq: float
    max_block_residual: float
    wall_ms: float
    clamped: bool


class BlockProblems:
    """What assemble_block_problems (blockform.py:48-86) returns here.

    The reference materialises per-block operators.  On a q == 1 lattice they
    reduce to the unary, lambda*w (or weight planes) and the block geometry,
    kept resident in HBM for the run loop's kernels (kind "int" / "float").
    Any other model / partition has kind "graph".  Indexing gives the
    reference's BlockProblem fields per block (u_hat, w_hat, d_hat, r_diag,
    c_rows, computed on demand) and the step-level API runs on the general
    graph path's device data (graph(), built on first use).
    """

    def __init__(self, model: EnergyModel, partition: Partition):
        import torch
        if model.n != partition.shape.n:
            raise ValueError("model and partition sizes differ")
        self.partition = partition
        self.model = model
        self.device = _device()
        self.lowering, self.kind, self.u = None, "graph", None
        for kind, lower in (("int", lower_lattice), ("float", lower_float)):
            try:
                self.lowering = lower(model, partition)
                self.kind = kind
                break
            except (NotImplementedError, NonSubmodularError):
                continue
        if self.lowering is not None:
            self.u = torch.as_tensor(self.lowering.u, device=self.device)
        self._graph = None

    def refresh_unary(self, model: EnergyModel, defer_check: bool = False) -> bool:
        """Take a new model that shares this one's weights, partition and lambda:
        upload its unary (the integer path converts and checks it on the device).
        False when the new unary does not fit this lowering.  With defer_check
        the integer check's verdict is read later (unary_confirmed), so the
        caller can enqueue the run behind the upload without a synchronisation;
        a lowering whose check then fails must be discarded."""
        import torch
        if model.weights is not self.model.weights or float(model.lam) != float(self.model.lam):
            return False
        if model is self.model:
            return True
        # pipelined pinned staging, or a direct DMA once the caller's buffer
        # repeats (hostio.UnaryUploader)
        if getattr(self, "_uploader", None) is None:
            from .hostio import UnaryUploader
            self._uploader = UnaryUploader(self.lowering.n, self.device)
        u64 = self._uploader.upload(model.unary)
        if self.kind == "int":
            bad = torch.zeros(1, dtype=torch.int32, device=self.device)
            _lib.check(_lib.lib().dope_unary_i32(u64.data_ptr(), u64.numel(), self.u.data_ptr(), bad.data_ptr(),
                                                 C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)),
                       "dope_unary_i32")
            self._pending_bad = bad
            if not defer_check and not self.unary_confirmed():
                return False
        elif self.kind == "float":
            self.u.copy_(u64)
        self.model = model
        self._graph = None
        return True

    def unary_confirmed(self) -> bool:
        """The device verdict of the last deferred unary check (synchronises)."""
        bad = getattr(self, "_pending_bad", None)
        self._pending_bad = None
        return bad is None or not bad.item()

    def run_state(self, mu, eps: float, config: "AdmmConfig"):
        """Device buffers for a run of this lowering, reused across runs with the
        same parameters (so the cached CUDA graph of the loop is reused too)."""
        key = (float(mu), float(eps), config.max_iters, config.warm_start, config.skip_clean, config.digests)
        last = getattr(self, "_run_owner", None)
        if last is not None and last() is not None:
            last()._detach()      # a live state of the previous run keeps its own copy
        if getattr(self, "_run_key", None) != key:
            self._run_dev = make_device_state(self, mu, eps, config.max_iters, config.warm_start,
                                              config.skip_clean, config.digests)
            self._run_key = key
        elif self._run_dev.trace_hash is not None:
            self._run_dev.trace_hash.zero_()
        return self._run_dev

    def graph(self):
        """The general graph path's device data (graphstep.GraphProblems)."""
        if self._graph is None:
            from .graphstep import GraphProblems
            self._graph = GraphProblems(self.model, self.partition)
        return self._graph

    def __len__(self) -> int:
        return self.partition.k

    def __getitem__(self, k: int):
        return self.graph()[k]

    def __iter__(self):
        return iter(self.graph())

    @property
    def lam(self) -> float:
        return float(self.model.lam)


class _FloatDeviceState:
    """Caller-owned device buffers of one float-weight run (dope_lattice_f)."""

    def __init__(self, problems: BlockProblems, mu: float, eps: float, max_iters: int,
                 warm_start: bool, skip_clean: bool, digests: bool = False):
        import torch
        low: FloatLowering = problems.lowering
        dev = problems.device
        n, K = low.n, low.K
        self.problems = problems
        self.max_iters = max_iters
        L = self.L = _lib.LatticeF()
        L.conn = low.conn
        L.dims[0], L.dims[1] = low.dims
        L.kpa[0], L.kpa[1] = low.kpa
        L.lam, L.mu, L.eps, L.qscale = low.lam, float(mu), float(eps), low.qscale
        L.max_iters, L.warm_start, L.skip_clean, L.fuse_multipliers = (
            max_iters, int(warm_start), int(skip_clean), 1)
        lb = _lib.lib()
        stride = lb.dope_f_resid_stride(C.byref(L))
        if stride <= 0:
            raise NotImplementedError(f"no float K1 variant for {low.dims}/{low.kpa}")
        f64 = torch.float64
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
        self.w = [t(p) for p in low.w]
        self.capq = [t(p) for p in low.capq]
        self.rdiag = t(low.rdiag)
        self.a = [torch.zeros(n, dtype=f64, device=dev) for _ in range(2)]
        self.y2 = [torch.full((n,), 0.5, dtype=f64, device=dev) for _ in range(3)]
        self.yhat = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.resid = torch.zeros(K * stride // 4, dtype=torch.int32, device=dev)
        # [0, K) re-solve flags, [K, 2K) solve epochs, [2K, 5K) y-buffer stamps,
        # [5K, 6K) last change of each block's iterate (clean-block pass)
        # [6K, 7K) pass of each block's interior energy from K1f (energy_prepass)
        self.dirty = torch.zeros(7 * K, dtype=torch.int32, device=dev)
        self.dirty[:K] = 1
        self.pe = torch.zeros(33 * K, dtype=f64, device=dev)   # [K, 33K): K1f's per-warp interior energy sums
        L.energy_prepass = int(os.environ.get("DOPE_F_EPRE", "1"))
        self.pr = torch.zeros(K, dtype=f64, device=dev)
        self.pf = torch.zeros(K, dtype=torch.int32, device=dev)
        self.state = torch.zeros(C.sizeof(_lib.RunState), dtype=torch.uint8, device=dev)
        self.tr_e = torch.zeros(max_iters, dtype=f64, device=dev)
        self.tr_rs = torch.zeros(max_iters, dtype=f64, device=dev)
        self.tr_mr = torch.zeros(max_iters, dtype=f64, device=dev)
        self.tr_cl = torch.zeros(max_iters, dtype=torch.int32, device=dev)
        L.u = problems.u.data_ptr()
        for i in range(4):
            L.w[i] = self.w[i].data_ptr()
            L.capq[i] = self.capq[i].data_ptr()
        L.rdiag = self.rdiag.data_ptr()
        L.a[0], L.a[1] = self.a[0].data_ptr(), self.a[1].data_ptr()
        for i in range(3):
            L.y[i] = self.y2[i].data_ptr()
        L.yhat = self.yhat.data_ptr()
        L.resid = self.resid.data_ptr()
        L.dirty = self.dirty.data_ptr()
        L.part_energy, L.part_ressq, L.part_flags = (self.pe.data_ptr(), self.pr.data_ptr(),
                                                     self.pf.data_ptr())
        L.state = self.state.data_ptr()
        L.trace_energy, L.trace_residual_sq = self.tr_e.data_ptr(), self.tr_rs.data_ptr()
        L.trace_max_residual, L.trace_clamped = self.tr_mr.data_ptr(), self.tr_cl.data_ptr()
        self.trace_hash = (torch.zeros(3 * max_iters + 2, dtype=torch.int64, device=dev)
                           if digests else None)
        if digests:
            L.trace_hash = self.trace_hash.data_ptr()
        _lib.check(lb.dope_f_check(C.byref(L)), "dope_f_check")

    _NAMES = {"dope_admm_init": "dope_f_admm_init", "dope_update_blocks": "dope_f_update_blocks",
              "dope_update_global": "dope_f_update_global",
              "dope_update_multipliers": "dope_f_update_multipliers",
              "dope_admm_run": "dope_f_admm_run", "dope_finish_run": "dope_f_finish_run"}

    def stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream(self.problems.device).cuda_stream)

    def call(self, name: str, *args, fuse: int | None = None):
        if fuse is not None:
            self.L.fuse_multipliers = fuse
        fname = self._NAMES[name]
        _lib.check(getattr(_lib.lib(), fname)(C.byref(self.L), *args, self.stream()), fname)

    def run_state(self) -> _lib.RunState:
        return _lib.RunState.from_buffer_copy(self.state.cpu().numpy().tobytes())

    def y2_current(self, rs=None):
        # float path stores y itself; expose 2*y for a uniform host view
        return self.y2[(self.run_state() if rs is None else rs).ycur] * 2.0

    def multipliers(self, rs=None):
        return self.a[(self.run_state() if rs is None else rs).parity]

    def binarize(self):
        import torch
        out = torch.empty(self.problems.lowering.n, dtype=torch.uint8, device=self.problems.device)
        _lib.check(_lib.lib().dope_f_binarize(C.byref(self.L), out.data_ptr(), self.stream()),
                   "dope_f_binarize")
        return out

    def raise_on_error(self, rs=None):
        rs = self.run_state() if rs is None else rs
        if rs.error:
            raise BlockSolveError(rs.error - 1, "push-relabel round limit exceeded")
        return rs


def make_device_state(problems: BlockProblems, mu: float, eps: float, max_iters: int,
                      warm_start: bool = True, skip_clean: bool = True, digests: bool = False):
    """Device buffers of one run for the lowering kind (int or float lattice).
    digests: audit mode, per-iteration state digests in .trace_hash."""
    if problems.kind == "float":
        return _FloatDeviceState(problems, mu, eps, max_iters, warm_start, skip_clean, digests)
    return _DeviceState(problems, int(mu), eps, max_iters, warm_start, skip_clean, digests)


def assemble_block_problems(model: EnergyModel, partition: Partition) -> BlockProblems:
    """blockform.assemble_block_problems (blockform.py:48-86): the device lowering."""
    return BlockProblems(model, partition)


_lowered: dict = {}


def _problems_for(model: EnergyModel, partition: Partition, defer_check: bool = False) -> BlockProblems:
    """assemble_block_problems, reused when the same weights / partition come
    back with new unaries (the serving loop of run(): the lattice checks and
    device buffers are kept, only the unary is uploaded)."""
    import weakref
    key = (id(model.weights), id(partition))
    hit = _lowered.get(key)
    if hit is not None and hit[0]() is model.weights and hit[1]() is partition:
        if hit[2].refresh_unary(model, defer_check):
            return hit[2]
    problems = BlockProblems(model, partition)
    drop = lambda _r, k=key: _lowered.pop(k, None)
    _lowered[key] = (weakref.ref(model.weights, drop), weakref.ref(partition, drop), problems)
    return problems


def _forget(problems: BlockProblems):
    for key, hit in list(_lowered.items()):
        if hit[2] is problems:
            _lowered.pop(key, None)


class _DeviceState:
    """Caller-owned device buffers of one run (include/dope_b200.h)."""

    def __init__(self, problems: BlockProblems, mu: int, eps: float, max_iters: int,
                 warm_start: bool, skip_clean: bool, digests: bool = False):
        import torch
        low = problems.lowering
        dev = problems.device
        n, K = low.n, low.K
        self.problems = problems
        self.max_iters = max_iters
        self.L = _lib.Lattice()
        L = self.L
        L.ndim = len(low.dims)
        L.conn = low.conn
        for ax in range(3):
            L.dims[ax] = low.dims[ax] if ax < len(low.dims) else 1
            L.kpa[ax] = low.kpa[ax] if ax < len(low.kpa) else 1
        L.lamw = low.lamw
        L.mu = mu
        L.eps = eps
        L.max_iters = max_iters
        L.warm_start = int(warm_start)
        L.skip_clean = int(skip_clean)
        L.fuse_multipliers = 1
        lb = _lib.lib()
        stride = lb.dope_resid_stride(C.byref(L))
        if stride <= 0:
            raise NotImplementedError(f"no K1 kernel variant for block box of {low.dims}/{low.kpa}")
        i32, u8 = torch.int32, torch.uint8
        # multipliers fit int16 (|a| <= t + 1, max_iters is capped below 32000);
        # 2y in {0, 1, 2} is one byte
        self.a = torch.zeros(n, dtype=torch.int16, device=dev)   # updated in place
        # y2 and yhat carry one ghost row (2D) / plane (3D) on each side (neighbour
        # shards; unused on a single GPU), the ABI points one unit into the allocation
        g = int(np.prod(low.dims[1:]))   # one ghost row (2D) / plane (3D) on each side
        self.ghost = g
        self.y2_full = [torch.ones(n + 2 * g, dtype=u8, device=dev) for _ in range(3)]
        self.y2 = [t[g:g + n] for t in self.y2_full]
        self.yhat_full = torch.zeros(n + 2 * g, dtype=u8, device=dev)
        self.yhat = self.yhat_full[g:g + n]
        self.agg = torch.zeros(4, dtype=torch.int64, device=dev)
        self.resid = torch.zeros(K * stride, dtype=u8, device=dev)
        # [0, K): re-solve flags; [K, 2K): iteration + 1 of each block's last solve;
        # [2K, 7K): y-buffer / iterate-change / energy-partial stamps of the
        # clean-block consensus passes; [7K, 9K): the solved-block list and slots;
        # [9K, 11K + 2): the run loop's dirty-block worklists; [11K + 2, 12K + 2):
        # finished-solve epochs (K1 / consensus overlap); [12K + 2, 16K + 8): the
        # consensus pass's tile-work queue
        self.dirty = torch.zeros(16 * K + 8, dtype=torch.int32, device=dev)
        self.dirty[:K] = 1
        sstride = int(lb.dope_scratch_stride(C.byref(L)))
        self.scratch = torch.empty(max(K * sstride, 16), dtype=u8, device=dev)
        self.pe = torch.zeros(K, dtype=torch.int64, device=dev)
        self.pu = torch.zeros(K, dtype=torch.int64, device=dev)
        self.pr = torch.zeros(K, dtype=torch.int64, device=dev)
        self.pf = torch.zeros(K, dtype=i32, device=dev)
        self.pc = torch.zeros(_lib.PART_CTA_LEN, dtype=torch.int64, device=dev)
        self.state = torch.zeros(C.sizeof(_lib.RunState), dtype=u8, device=dev)
        self.tr_e = torch.zeros(max_iters, dtype=torch.int64, device=dev)
        self.tr_rs = torch.zeros(max_iters, dtype=torch.float64, device=dev)
        self.tr_mr = torch.zeros(max_iters, dtype=torch.float64, device=dev)
        self.tr_cl = torch.zeros(max_iters, dtype=i32, device=dev)
        L.u = problems.u.data_ptr()
        L.a = self.a.data_ptr()
        for i in range(3):
            L.y2[i] = self.y2[i].data_ptr()
        L.yhat = self.yhat.data_ptr()
        L.resid = self.resid.data_ptr()
        L.dirty = self.dirty.data_ptr()
        L.scratch = self.scratch.data_ptr()
        L.part_energy = self.pe.data_ptr()
        L.part_unary = self.pu.data_ptr()
        L.part_ressq = self.pr.data_ptr()
        L.part_flags = self.pf.data_ptr()
        L.part_cta = self.pc.data_ptr()
        L.state = self.state.data_ptr()
        L.trace_energy = self.tr_e.data_ptr()
        L.trace_residual_sq = self.tr_rs.data_ptr()
        L.trace_max_residual = self.tr_mr.data_ptr()
        L.trace_clamped = self.tr_cl.data_ptr()
        L.agg = self.agg.data_ptr()
        # audit mode: per-iteration (yhat, 2y, a) digests (dope_lattice.trace_hash)
        self.trace_hash = (torch.zeros(3 * max_iters + 2, dtype=torch.int64, device=dev)
                           if digests else None)
        if digests:
            L.trace_hash = self.trace_hash.data_ptr()
        _lib.check(lb.dope_lattice_check(C.byref(L)), "dope_lattice_check")

    def stream(self):
        import torch
        return C.c_void_p(torch.cuda.current_stream(self.problems.device).cuda_stream)

    def call(self, name: str, *args, fuse: int | None = None):
        if fuse is not None:
            self.L.fuse_multipliers = fuse
        fn = getattr(_lib.lib(), name)
        _lib.check(fn(C.byref(self.L), *args, self.stream()), name)

    def run_state(self) -> _lib.RunState:
        raw = self.state.cpu().numpy().tobytes()
        return _lib.RunState.from_buffer_copy(raw)

    def y2_current(self, rs=None):
        return self.y2[(self.run_state() if rs is None else rs).ycur]

    def multipliers(self, rs=None):
        return self.a

    def binarize(self):
        import torch
        out = torch.empty(self.problems.lowering.n, dtype=torch.uint8, device=self.problems.device)
        lb = _lib.lib()
        _lib.check(lb.dope_binarize(C.byref(self.L), out.data_ptr(), self.stream()), "dope_binarize")
        return out

    def raise_on_error(self, rs=None):
        rs = self.run_state() if rs is None else rs
        if rs.error == -1:
            raise OverflowError("a multiplier left the int16 range (|a| > 32000); "
                                "the run exceeded the iteration range the compressed state holds")
        if rs.error:
            raise BlockSolveError(rs.error - 1, "push-relabel round limit exceeded")
        return rs

    def reset_unary(self):
        """Recompute the running unary term sum u*y2 after a host write of y."""
        import torch
        off = _lib.RunState.unary2.offset
        val = (self.problems.u.to(torch.int64) * self.y2_current().to(torch.int64)).sum()
        self.state[off:off + 8].view(torch.int64).copy_(val.reshape(1))


class AdmmState:
    """Mutable state of one run (admm.py:87-99), with the reference's fields.

    y, block_labels and multipliers are host numpy arrays (lists of per-block
    arrays) exactly like the reference's dataclass: in-place edits such as
    ``state.multipliers[k] += d`` or ``state.y = v`` are what the next step
    call sees -- every step function uploads the state it reads and downloads
    what it writes (the step API's device kernels are csrc/dope_gstep.cu).  A
    state returned by run() keeps them on the device and materialises each one
    on first access (a 4096^2 run never copies 4096 block lists otherwise).
    """

    def __init__(self, y=None, block_labels=None, multipliers=None, mu: float = 0.0,
                 iteration: int = 0, converged: bool = False, best_iteration: int = 0,
                 trace=None, clamped_last: bool = False, partition: Partition | None = None):
        self._y, self._block_labels, self._multipliers = y, block_labels, multipliers
        self.mu = float(mu)
        self.iteration = iteration
        self.converged = converged
        self.best_iteration = best_iteration
        self.trace: list = [] if trace is None else trace
        self.clamped_last = clamped_last
        self.partition = partition
        self.digests = None        # (iterations, 3) uint64 when AdmmConfig.digests
        self._src = None           # device source of the fields not yet materialised

    # -- construction from a finished device run --------------------------------
    @classmethod
    def from_lattice(cls, partition: Partition, dev, mu: float, rs=None) -> "AdmmState":
        """Fields live in a lattice run's device buffers (global layout, q == 1);
        rs = the run state read back at the end of the run."""
        st = cls(mu=mu, partition=partition)
        st._src = ("lattice", dev)
        st._rs = rs
        return st

    def _detach(self):
        """Snapshot a lattice run's fields before its device buffers are reused by
        the next run of the same problems: device-to-device copies of the
        compressed state (2y bytes, labels, multipliers), still materialised
        lazily.  Enqueued without a synchronisation (the buffer indices come
        from the run state read back when the run ended)."""
        if self._src is not None and self._src[0] == "lattice":
            dev, rs = self._src[1], getattr(self, "_rs", None)
            self._src = ("lattice_copy", (dev.y2_current(rs).clone(), dev.yhat.clone(),
                                          dev.multipliers(rs).clone()))

    @classmethod
    def from_device(cls, partition: Partition, y, yhat_cat, a_cat, layout, mu: float) -> "AdmmState":
        """Fields live in the general graph path's entry-indexed device buffers."""
        st = cls(mu=mu, partition=partition)
        st._src = ("entries", (y, yhat_cat, a_cat, layout))
        return st

    def _entries(self):
        from .graphstep import layout
        return layout(self.partition)

    def _fetch(self, what: str):
        kind, src = self._src
        if kind == "lattice_copy":
            y2, yhat, a = src
            if what == "y":
                return y2.double().div_(2.0).cpu().numpy()
            lay = self._entries()
            if what == "block_labels":
                return lay.split(yhat.cpu().numpy()[lay.ent_pix].astype(np.int8))
            return lay.split(a.double().cpu().numpy()[lay.ent_pix])
        if kind == "lattice":
            dev = src
            if what == "y":
                return dev.y2_current().double().div_(2.0).cpu().numpy()
            lay = self._entries()
            if what == "block_labels":
                return lay.split(dev.yhat.cpu().numpy()[lay.ent_pix].astype(np.int8))
            return lay.split(dev.multipliers().double().cpu().numpy()[lay.ent_pix])
        y, yhat, a, lay = src
        if what == "y":
            return y.cpu().numpy().copy()
        if what == "block_labels":
            return lay.split(yhat[:lay.M].cpu().numpy().astype(np.int8))
        return lay.split(a[:lay.M].cpu().numpy().copy())

    @property
    def y(self) -> np.ndarray:
        if self._y is None and self._src is not None:
            self._y = self._fetch("y")
        return self._y

    @y.setter
    def y(self, value):
        self._y = np.asarray(value, dtype=np.float64)

    @property
    def block_labels(self) -> list:
        if self._block_labels is None and self._src is not None:
            self._block_labels = self._fetch("block_labels")
        return self._block_labels

    @block_labels.setter
    def block_labels(self, value):
        self._block_labels = list(value)

    @property
    def multipliers(self) -> list:
        if self._multipliers is None and self._src is not None:
            self._multipliers = self._fetch("multipliers")
        return self._multipliers

    @multipliers.setter
    def multipliers(self, value):
        self._multipliers = list(value)

    # -- global-layout helpers (non-overlapping partitions) -----------------------
    def _to_global(self, per_block, dtype) -> np.ndarray:
        lay = self._entries()
        if lay.M != lay.n:
            raise ValueError("global layout needs a non-overlapping partition")
        out = np.empty(lay.n, dtype=dtype)
        out[lay.ent_pix] = lay.join(per_block, dtype, "vectors")
        return out

    def labels_global(self) -> np.ndarray:
        """Current block labels (yhat) scattered to global layout."""
        if self._block_labels is None and self._src is not None and self._src[0] == "lattice":
            return self._src[1].yhat.cpu().numpy().astype(np.int8)
        if self._block_labels is None and self._src is not None and self._src[0] == "lattice_copy":
            return self._src[1][1].cpu().numpy().astype(np.int8)
        return self._to_global(self.block_labels, np.int8)

    def multipliers_global(self) -> np.ndarray:
        if self._multipliers is None and self._src is not None and self._src[0] == "lattice":
            return self._src[1].multipliers().double().cpu().numpy()
        if self._multipliers is None and self._src is not None and self._src[0] == "lattice_copy":
            return self._src[1][2].double().cpu().numpy()
        return self._to_global(self.multipliers, np.float64)


def init_state(partition: Partition, mu0: float) -> AdmmState:
    """y = 1/2, zero multipliers, zero block labels (admm.py:100-110)."""
    n = partition.shape.n
    return AdmmState(np.full(n, 0.5), [np.zeros(b.size, dtype=np.int8) for b in partition.blocks],
                     [np.zeros(b.size) for b in partition.blocks], float(mu0), partition=partition)


# ---------------------------------------------------------------------------
# Step-level API (admm.py:113-204) on the general graph path
# ---------------------------------------------------------------------------

def _graph(problems):
    from .graphstep import GraphProblems
    if isinstance(problems, GraphProblems):
        return problems
    if isinstance(problems, BlockProblems):
        return problems.graph()
    raise TypeError("problems must come from assemble_block_problems")


def _dev_vec(v, dtype, dev):
    import torch
    return torch.as_tensor(np.ascontiguousarray(v, dtype=dtype), device=dev)


def _dev_entries(gp_layout, per_block, dtype, what):
    import torch
    cat = gp_layout.join(per_block, dtype, what)
    t = torch.zeros(max(gp_layout.M, 1), dtype=torch.uint8 if dtype == np.uint8 else torch.float64,
                    device=gp_layout.device)
    if gp_layout.M:
        t[:gp_layout.M] = torch.as_tensor(cat, device=gp_layout.device)
    return t


def _lattice_blocks(state: AdmmState, problems: BlockProblems, lam: float, config: AdmmConfig):
    """update_blocks on the integer lattice K1 (dope_update_blocks) when the
    state is one the kernel represents exactly: y in {0, 1/2, 1}, integer
    multipliers within int16, an integer mu dividing lambda*w (q == 1).
    Returns the per-block labels, or None when the state does not qualify."""
    import torch
    low = problems.lowering
    mu = state.mu
    if (problems.kind != "int" or config.solver.kind != "maxflow" or float(lam) != problems.lam
            or not mu > 0 or mu != round(mu) or low.lamw % int(round(mu))):
        return None
    y2 = 2.0 * np.asarray(state.y, dtype=np.float64)
    if y2.shape != (low.n,) or not np.all(np.isin(y2, (0.0, 1.0, 2.0))):
        return None
    from .graphstep import layout
    lay = layout(problems.partition)
    a = np.empty(low.n)
    a[lay.ent_pix] = lay.join(state.multipliers, np.float64, "multipliers")
    if not np.all(a == np.round(a)) or np.abs(a).max(initial=0) > 32000:
        return None
    dev = getattr(problems, "_step_dev", None)
    if dev is None:
        dev = problems._step_dev = _DeviceState(problems, int(round(mu)), 0.0, 1, True, False)
        dev.call("dope_admm_init")
    dev.L.mu = int(round(mu))
    dev.y2_current().copy_(torch.as_tensor(y2.astype(np.uint8), device=problems.device))
    dev.a.copy_(torch.as_tensor(a.astype(np.int16), device=problems.device))
    dev.dirty[:low.K].fill_(1)
    dev.call("dope_update_blocks")
    dev.raise_on_error()
    return lay.split(dev.yhat.cpu().numpy()[lay.ent_pix].astype(np.int8))


def update_blocks(state: AdmmState, problems, lam: float, config: AdmmConfig) -> AdmmState:
    """Re-solve every block against the current y (admm.py:113-133): block
    objectives and block min cuts (one CTA per block) on the device -- the
    integer lattice K1 when the state is one it represents exactly, else the
    general graph path."""
    if isinstance(problems, BlockProblems):
        labels = _lattice_blocks(state, problems, lam, config)
        if labels is not None:
            state.block_labels = labels
            return state
    gp = _graph(problems)
    lay = gp.layout
    y = _dev_vec(state.y, np.float64, gp.device)
    if y.shape != (lay.n,):
        raise ValueError(f"y has shape {tuple(y.shape)}, expected ({lay.n},)")
    a = _dev_entries(lay, state.multipliers, np.float64, "multipliers")
    lin = gp.objective(y, a, state.mu, lam)
    labels = gp.solve(lin, lam, config.solver.kind)
    state.block_labels = lay.split(labels[:lay.M].cpu().numpy().astype(np.int8))
    return state


def solve_global(problems, partition: Partition, block_labels: list, multipliers: list, mu: float,
                 lam: float) -> np.ndarray:
    """Unclamped closed-form global minimiser (admm.py:136-151) on the device."""
    gp = _graph(problems)
    lay = gp.layout
    yhat = _dev_entries(lay, [np.asarray(b) for b in block_labels], np.uint8, "labels")
    a = _dev_entries(lay, multipliers, np.float64, "multipliers")
    y, _ = gp.solve_global(yhat, a, mu, lam, clamp=False)
    return y.cpu().numpy()


def consensus_objective(problems, partition: Partition, block_labels: list, multipliers: list,
                        mu: float, lam: float, y) -> float:
    """lam sum_k yhat_k' (C_k + R_k S_k) y + mu/2 sum_k ||S_k y - (yhat_k + a_k)||^2
    (admm.py:154-169): per-block terms on the device, summed in block order."""
    gp = _graph(problems)
    lay = gp.layout
    yhat = _dev_entries(lay, [np.asarray(b) for b in block_labels], np.uint8, "labels")
    a = _dev_entries(lay, multipliers, np.float64, "multipliers")
    parts = gp.consensus_parts(yhat, a, _dev_vec(y, np.float64, gp.device))
    total = 0.0
    for c, p in parts:
        total += lam * float(c)
        total += 0.5 * mu * float(p)
    return total


def update_global(state: AdmmState, problems, partition: Partition, lam: float) -> AdmmState:
    """Closed-form global step, clamped into [0, 1] (admm.py:172-180)."""
    gp = _graph(problems)
    lay = gp.layout
    yhat = _dev_entries(lay, [np.asarray(b) for b in state.block_labels], np.uint8, "labels")
    a = _dev_entries(lay, state.multipliers, np.float64, "multipliers")
    y, flag = gp.solve_global(yhat, a, state.mu, lam, clamp=True)
    state.clamped_last = bool(flag.item())
    state.y = y.cpu().numpy()
    return state


def update_multipliers(state: AdmmState, partition: Partition, mu_fact: float) -> AdmmState:
    """a_k += yhat_k - S_k y, then mu *= mu_fact (admm.py:183-190), on the device."""
    from .graphstep import layout, update_multipliers_dev
    lay = layout(partition)
    yhat = _dev_entries(lay, [np.asarray(b) for b in state.block_labels], np.uint8, "labels")
    a = _dev_entries(lay, state.multipliers, np.float64, "multipliers")
    update_multipliers_dev(lay, yhat, _dev_vec(state.y, np.float64, lay.device), a)
    state.multipliers = lay.split(a[:lay.M].cpu().numpy())
    state.mu *= mu_fact
    return state


def block_residuals(state: AdmmState, partition: Partition) -> np.ndarray:
    """Per-block ||yhat_k - S_k y|| (admm.py:193-199), on the device."""
    from .graphstep import layout, residuals_sq
    lay = layout(partition)
    yhat = _dev_entries(lay, [np.asarray(b) for b in state.block_labels], np.uint8, "labels")
    ss = residuals_sq(lay, yhat, _dev_vec(state.y, np.float64, lay.device))
    return np.sqrt(ss.cpu().numpy())


def binarize(y) -> np.ndarray:
    """y >= 1/2 -> 1, exact ties to 1 (admm.py:202-204)."""
    return (np.asarray(y) >= 0.5).astype(np.int8)


# ---------------------------------------------------------------------------
# run
# ---------------------------------------------------------------------------

class _StaleUnary(Exception):
    """A deferred unary check failed: the cached integer lowering cannot take
    this model's unary (run() re-lowers it from scratch)."""


def _run_lattice(model, partition, config, problems) -> tuple:
    import torch
    mu0 = config.resolved_mu0(partition.shape.ndim)
    eps = config.resolved_eps(partition)
    if problems.kind == "int" and (mu0 != round(mu0) or problems.lowering.lamw % int(round(mu0)) != 0):
        if not problems.unary_confirmed():
            raise _StaleUnary()
        raise NotImplementedError("the integer lattice path needs an integer mu dividing lambda*w")
    dev = problems.run_state(mu0, eps, config)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    dev.call("dope_admm_init")
    dev.call("dope_admm_run", config.max_iters, int(config.use_graph), fuse=1)
    dev.call("dope_finish_run")
    end.record()
    # one batch of D2H copies (labels of the best / final iterate, run state,
    # trace) and one synchronisation
    if getattr(problems, "_downloader", None) is None:
        from .hostio import LabelDownloader
        problems._downloader = LabelDownloader(problems.lowering.n)
    small = {"state": dev.state, "e": dev.tr_e, "rs": dev.tr_rs, "mr": dev.tr_mr, "cl": dev.tr_cl}
    if dev.trace_hash is not None:
        small["hash"] = dev.trace_hash
    problems._downloader.enqueue(dev.binarize(), small)
    labels, host = problems._downloader.wait()
    if not problems.unary_confirmed():
        raise _StaleUnary()
    total_ms = start.elapsed_time(end)
    rs = _lib.RunState.from_buffer_copy(host["state"].tobytes())
    dev.raise_on_error(rs)
    it = rs.iteration
    e, r2, mr, cl = host["e"][:it], host["rs"][:it], host["mr"][:it], host["cl"][:it]
    per = total_ms / max(it, 1)   # one graph launch: the per-iteration average
    state = AdmmState.from_lattice(partition, dev, mu0, rs)
    import weakref
    problems._run_owner = weakref.ref(state)
    mu = mu0
    for t in range(it):
        state.trace.append(TraceRecord(t + 1, mu, float(e[t]), float(r2[t]), float(mr[t]), per, bool(cl[t])))
        mu *= config.mu_fact
    state.mu = mu
    state.iteration = it
    state.converged = bool(rs.converged)
    state.best_iteration = int(rs.best_iteration)
    state.clamped_last = bool(cl[it - 1]) if it else False
    if dev.trace_hash is not None:
        state.digests = host["hash"][:3 * it].view(np.uint64).reshape(it, 3)
    return labels, state


_max_counts: dict = {}


def _max_count(partition: Partition) -> int:
    """max q over pixels, computed once per partition object (an O(n) scan of
    partition.counts would otherwise cost ~3.5 ms per run() at 4096^2)."""
    import weakref
    key = id(partition)
    hit = _max_counts.get(key)
    if hit is not None and hit[0]() is partition:
        return hit[1]
    q = int(partition.counts.max()) if partition.counts.size else 1
    _max_counts[key] = (weakref.ref(partition, lambda _r, k=key: _max_counts.pop(k, None)), q)
    return q


def run(model: EnergyModel, partition: Partition, config: AdmmConfig,
        problems: BlockProblems | None = None):
    """Full distributed minimisation on the GPU (admm.py:207-252).

    Returns (y_binary, state) with the reference's semantics: the best
    relaxed-energy iterate when max_iters runs out (state.y is then that
    iterate), the final iterate when converged.  Dispatch, fastest first:
    the exact integer lattice kernels (q == 1, integer u and lambda*w, integer
    mu dividing it, mu_fact == 1), the float lattice kernels (2D 4/8-connected,
    q == 1, mu_fact == 1), the 2D lattice overlap / mu-schedule kernels
    (dope_general), and the general graph path for everything else (any pair
    set, 3D overlap, any schedule).  All of them run on the device.
    """
    if config.solver.kind == "icm":
        raise NotImplementedError("the ICM block solver has no B200 kernel (out of scope)")
    if problems is not None and not isinstance(problems, BlockProblems):
        from .graphstep import GraphProblems, run_graph
        if isinstance(problems, GraphProblems):
            return run_graph(model, partition, config, problems)
        raise TypeError("problems must come from assemble_block_problems")
    overlap = partition.overlap_pct != 0 or _max_count(partition) > 1
    lattice_ok = config.solver.kind == "maxflow"
    if lattice_ok and not overlap and config.mu_fact == 1.0:
        cached = problems is None
        if cached:
            problems = _problems_for(model, partition, defer_check=True)
        if problems.kind in ("int", "float"):
            try:
                return _run_lattice(model, partition, config, problems)
            except NotImplementedError:
                pass
            except _StaleUnary:
                # the reused integer lowering cannot hold this unary: lower anew
                _forget(problems)
                return run(model, partition, config)
    if lattice_ok and partition.shape.ndim == 2:
        from .general import lower_general, run_general
        try:
            lower_general(model, partition)
        except NotImplementedError:
            pass
        else:
            return run_general(model, partition, config, use_graph=config.use_graph)
    from .graphstep import run_graph
    return run_graph(model, partition, config, problems.graph() if problems is not None else None)
