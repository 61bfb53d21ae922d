"""Consensus (ADMM) loop on the B200: API mirror of reference admm.py:27-310.

Same names, arguments, side effects on AdmmState and error types as the
reference; the work runs in libdope_b200.so through the C ABI
(include/dope_b200.h):

  update_blocks      -> dope_update_blocks     (K1, one CTA per sub-region)
  update_global      -> dope_update_global     (K2: y, clamp, residual and
                                                energy partials)
  update_multipliers -> dope_update_multipliers
  block_residuals    <- K2's per-block partials
  run                -> dope_admm_init + dope_admm_run (K1, K2+multipliers,
                        K3 per iteration, CUDA graph, no host sync inside the
                        loop) + dope_finish_run

State lives on the device; AdmmState.y / block_labels / multipliers
materialize host arrays on access.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .energy import EnergyModel
from .lowering import FloatLowering, LatticeLowering, lower_float, lower_lattice
from .partition import Partition


class BlockSolveError(RuntimeError):
    """A block solver failed; carries the block id (admm.py:85-90)."""

    def __init__(self, block_id: int, cause):
        super().__init__(f"solver failed on block {block_id}: {cause}")
        self.block_id = block_id


def _device():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the DOPE B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class BlockSolverKind:
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


@dataclass
class AdmmConfig:
    """Loop parameters (admm.py:93-129) plus B200 execution options."""

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
    """Device-lowered block problems: what assemble_block_problems returns here.

    The reference materializes per-block operators (blockform.py:216-254);
    on the q == 1 lattice they reduce to the unary, lambda*w and the block
    geometry, kept resident in HBM.
    """

    def __init__(self, model: EnergyModel, partition: Partition):
        import torch
        try:
            self.lowering = lower_lattice(model, partition)
            self.kind = "int"
        except NotImplementedError:
            # not an integer 4/6-connected constant-weight lattice: the float path (2D,
            # 4/8-connected, any non-negative weights); it raises if that fails too
            self.lowering = lower_float(model, partition)
            self.kind = "float"
        self.partition = partition
        self.model = model
        self.device = _device()
        self.u = torch.as_tensor(self.lowering.u, device=self.device)

    def __len__(self) -> int:
        return self.lowering.K

    @property
    def lam(self) -> float:
        return self.lowering.lam


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
        self.dirty = torch.ones(K, dtype=torch.int32, device=dev)
        self.pe = torch.zeros(K, dtype=f64, device=dev)
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

    def y2_current(self):
        # float path stores y itself; expose 2*y for a uniform host view
        return self.y2[self.run_state().ycur] * 2.0

    def multipliers(self):
        return self.a[self.run_state().parity]

    def binarize(self):
        import torch
        out = torch.empty(self.problems.lowering.n, dtype=torch.uint8, device=self.problems.device)
        _lib.check(_lib.lib().dope_f_binarize(C.byref(self.L), out.data_ptr(), self.stream()),
                   "dope_f_binarize")
        return out

    def raise_on_error(self):
        rs = self.run_state()
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
    return BlockProblems(model, partition)


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
        # clean-block consensus passes; [7K, 9K): the solved-block list and slots
        self.dirty = torch.zeros(9 * K, dtype=torch.int32, device=dev)
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

    def y2_current(self):
        return self.y2[self.run_state().ycur]

    def multipliers(self):
        return self.a

    def binarize(self):
        import torch
        out = torch.empty(self.problems.lowering.n, dtype=torch.uint8, device=self.problems.device)
        lb = _lib.lib()
        _lib.check(lb.dope_binarize(C.byref(self.L), out.data_ptr(), self.stream()), "dope_binarize")
        return out

    def raise_on_error(self):
        rs = self.run_state()
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
    """Mutable state of one run (admm.py:145-157), resident on the device."""

    def __init__(self, partition: Partition, mu: float):
        self.partition = partition
        self.mu = float(mu)
        self.iteration = 0
        self.converged = False
        self.best_iteration = 0
        self.clamped_last = False
        self.trace: list = []
        self.digests = None     # (iterations, 3) uint64 when AdmmConfig.digests
        self._dev: _DeviceState | None = None
        self._n = partition.shape.n

    # -- device binding ---------------------------------------------------
    def _bind(self, problems: BlockProblems, config: AdmmConfig, max_iters: int | None = None,
              eps: float = 0.0) -> _DeviceState:
        if self._dev is not None and self._dev.problems is problems:
            return self._dev
        mu = self.mu
        if problems.kind == "float":
            self._dev = _FloatDeviceState(problems, mu, eps, max_iters or config.max_iters,
                                          config.warm_start, config.skip_clean, config.digests)
            self._dev.call("dope_admm_init")
            return self._dev
        if mu != round(mu) or mu <= 0:
            raise NotImplementedError("the integer lattice path needs an integer mu")
        if problems.lowering.lamw % int(mu) != 0:
            raise NotImplementedError("the integer lattice path needs lambda*w divisible by mu")
        self._dev = _DeviceState(problems, int(mu), eps, max_iters or config.max_iters,
                                 config.warm_start, config.skip_clean, config.digests)
        self._dev.call("dope_admm_init")
        return self._dev

    # -- host views (reference attribute names) ---------------------------
    @property
    def y(self) -> np.ndarray:
        if self._dev is None:
            return np.full(self._n, 0.5)
        return self._dev.y2_current().double().div_(2.0).cpu().numpy()

    @y.setter
    def y(self, value):
        if self._dev is None:
            raise RuntimeError("bind the state to problems before assigning y")
        import torch
        v = np.asarray(value, dtype=np.float64)
        if v.shape != (self._n,) or (not isinstance(self._dev, _FloatDeviceState)
                                     and not np.all(np.isin(v, (0.0, 0.5, 1.0)))):
            raise NotImplementedError("the integer lattice path holds y in {0, 1/2, 1}")
        if isinstance(self._dev, _FloatDeviceState):
            self._dev.y2[self._dev.run_state().ycur].copy_(torch.as_tensor(v))
        else:
            self._dev.y2_current().copy_(torch.as_tensor((2 * v).astype(np.uint8)))
            self._dev.reset_unary()
        K = self._dev.problems.lowering.K
        self._dev.dirty[:K].fill_(1)
        if self._dev.dirty.numel() > 2 * K:   # y buffers rewritten: no stamp holds
            self._dev.dirty[2 * K:].zero_()

    def _global_to_blocks(self, vec: np.ndarray, dtype) -> list:
        out = []
        for b in self.partition.blocks:
            sl = tuple(slice(lo, hi) for lo, hi in b.extent)
            out.append(vec.reshape(self.partition.shape.dims)[sl].ravel().astype(dtype))
        return out

    @property
    def block_labels(self) -> list:
        if self._dev is None:
            return [np.zeros(b.size if b.pixels.size else int(np.prod([h - l for l, h in b.extent])),
                             dtype=np.int8) for b in self.partition.blocks]
        return self._global_to_blocks(self._dev.yhat.cpu().numpy(), np.int8)

    @property
    def multipliers(self) -> list:
        return self._global_to_blocks(self.multipliers_global(), np.float64)

    def multipliers_global(self) -> np.ndarray:
        if self._dev is None:
            return np.zeros(self._n)
        return self._dev.multipliers().double().cpu().numpy()

    def labels_global(self) -> np.ndarray:
        """Current block labels (yhat) in global layout."""
        return self._dev.yhat.cpu().numpy().astype(np.int8)


def init_state(partition: Partition, mu0: float) -> AdmmState:
    """y = 1/2, zero multipliers, zero block labels (admm.py:160-168)."""
    return AdmmState(partition, mu0)


def _check_lam(problems: BlockProblems, lam: float):
    if float(lam) != problems.lam:
        raise ValueError("lam differs from the lowered model's lambda")


def update_blocks(state: AdmmState, problems: BlockProblems, lam: float,
                  config: AdmmConfig) -> AdmmState:
    """Re-solve every (dirty) block on the GPU (admm.py:171-191)."""
    if config.solver.kind != "maxflow":
        raise NotImplementedError("only the max-flow block solver has a B200 kernel")
    _check_lam(problems, lam)
    dev = state._bind(problems, config)
    dev.call("dope_update_blocks")
    dev.raise_on_error()
    return state


def update_global(state: AdmmState, problems: BlockProblems, partition: Partition,
                  lam: float) -> AdmmState:
    """Closed-form global step, clamped into [0, 1] (admm.py:230-238)."""
    _check_lam(problems, lam)
    dev = state._bind(problems, AdmmConfig())
    dev.call("dope_update_global", fuse=0)
    # the step kernels do not keep the clean-block stamps: none holds any more
    dev.dirty[2 * len(problems):].zero_()
    state.clamped_last = bool(dev.pf.any().item())
    return state


def update_multipliers(state: AdmmState, partition: Partition, mu_fact: float) -> AdmmState:
    """a_k += yhat_k - S_k y, then mu *= mu_fact (admm.py:241-248)."""
    if state._dev is None:
        raise RuntimeError("state is not bound to device problems")
    if mu_fact != 1.0:
        raise NotImplementedError("the B200 path keeps mu fixed (mu_fact == 1)")
    state._dev.call("dope_update_multipliers")
    state.mu *= mu_fact
    return state


def block_residuals(state: AdmmState, partition: Partition) -> np.ndarray:
    """Per-block ||yhat_k - S_k y|| (admm.py:251-257), from the consensus partials."""
    if state._dev is None:
        raise RuntimeError("state is not bound to device problems")
    ss = state._dev.pr.cpu().numpy()
    return np.sqrt(ss.astype(np.float64))


def binarize(y) -> np.ndarray:
    return (np.asarray(y) >= 0.5).astype(np.int8)


def run(model: EnergyModel, partition: Partition, config: AdmmConfig,
        problems: BlockProblems | None = None):
    """Full distributed minimization on the GPU (admm.py:265-310).

    Returns (y_binary, state) with the reference's semantics: best relaxed
    energy iterate when max_iters runs out (state.y is then that iterate),
    the final iterate when converged.
    """
    import torch
    if config.solver.kind != "maxflow":
        raise NotImplementedError("only the max-flow block solver has a B200 kernel")
    overlap = partition.overlap_pct != 0 or bool(partition.counts.size and int(partition.counts.max()) > 1)
    if overlap or config.mu_fact != 1.0:
        # overlapping partitions / growing mu: the general path
        from .general import run_general
        return run_general(model, partition, config, use_graph=config.use_graph)
    if problems is None:
        problems = assemble_block_problems(model, partition)
    mu0 = config.resolved_mu0(partition.shape.ndim)
    eps = config.resolved_eps(partition)
    if problems.kind != "float" and partition.shape.ndim == 2 and (
            mu0 != round(mu0) or problems.lowering.lamw % int(round(mu0)) != 0):
        # the exact integer path needs mu | lambda*w; otherwise the general path
        from .general import run_general
        return run_general(model, partition, config, use_graph=config.use_graph)
    state = init_state(partition, mu0)
    dev = state._bind(problems, config, config.max_iters, eps)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    dev.call("dope_admm_run", config.max_iters, int(config.use_graph), fuse=1)
    dev.call("dope_finish_run")
    end.record()
    end.synchronize()
    total_ms = start.elapsed_time(end)
    rs = dev.raise_on_error()
    it = rs.iteration
    e = dev.tr_e[:it].cpu().numpy()
    r2 = dev.tr_rs[:it].cpu().numpy()
    mr = dev.tr_mr[:it].cpu().numpy()
    cl = dev.tr_cl[:it].cpu().numpy()
    per = total_ms / max(it, 1)
    mu = mu0
    for t in range(it):
        state.trace.append(TraceRecord(t + 1, mu, float(e[t]), float(r2[t]), float(mr[t]),
                                       per, bool(cl[t])))
        mu *= config.mu_fact
    state.mu = mu
    state.iteration = it
    state.converged = bool(rs.converged)
    state.best_iteration = int(rs.best_iteration)
    state.clamped_last = bool(cl[it - 1]) if it else False
    if dev.trace_hash is not None:
        state.digests = dev.trace_hash[:3 * it].cpu().numpy().view(np.uint64).reshape(it, 3)
    labels = dev.binarize().to(torch.int8).cpu().numpy()
    return labels, state
