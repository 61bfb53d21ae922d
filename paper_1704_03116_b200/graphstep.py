"""General graph path on the device: the ADMM step functions for ANY pairwise
model on ANY box partition (csrc/dope_gstep.cu, dope_bk_maxflow_batch).

The lattice kernels hold the benchmarked configurations; this module runs
whatever they cannot represent -- arbitrary SparseWeights pair sets (e.g. the
kernel-3/5/7 windows of build_potts_weights, random graphs), 3D overlapping
partitions, non-integer mu on integer models, blocks beyond the lattice
kernels' boxes -- and backs the reference's step-level API (admm.py:113-199:
update_blocks, solve_global, consensus_objective, update_global,
update_multipliers, block_residuals) and evaluate_energy (energy.py:187-194).
All arithmetic is float64 on the device, like the reference; with power-of-two
block counts and integer u / w / mu every value is a dyadic rational, hence
exact, and the min cuts (labels = the sink-reachable set, the reference's BK
sink tree) are bit-identical to the reference.

Layout ("entries"): block k's pixels, ascending (partition.py:52-59), are
entries blk_ptr[k] .. blk_ptr[k+1]; every pixel lists the entries holding it.
Block-local vectors (labels, multipliers, linear terms) are entry-indexed and
split into the reference's per-block lists on the host.
"""
from __future__ import annotations

import ctypes as C
import math
import weakref

import numpy as np

from . import _lib
from .energy import EnergyModel, NonSubmodularError
from .partition import Partition, box_pixels

EXHAUSTIVE_MAX_VARS = 24   # solvers.py:22

_layouts: dict = {}
_models: dict = {}


def _device():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the DOPE B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream(dev):
    import torch
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _cached(table: dict, obj, make):
    """Per-object cache that dies with the object (models / partitions hold arrays
    and are not hashable)."""
    key = id(obj)
    hit = table.get(key)
    if hit is not None and hit[0]() is obj:
        return hit[1]
    val = make()
    table[key] = (weakref.ref(obj, lambda _r, k=key: table.pop(k, None)), val)
    return val


class PartitionLayout:
    """Device entry layout of one partition (cached per Partition object)."""

    def __init__(self, partition: Partition, device):
        import torch
        self.partition = partition
        self.device = device
        shape = partition.shape
        self.n, self.K = shape.n, partition.k
        pix = [b.pixels if b.pixels.size == b.size else box_pixels(shape, b.extent)
               for b in partition.blocks]
        self.sizes = np.array([p.size for p in pix], dtype=np.int64)
        self.blk_ptr = np.zeros(self.K + 1, dtype=np.int64)
        np.cumsum(self.sizes, out=self.blk_ptr[1:])
        self.M = int(self.blk_ptr[-1])
        self.ent_pix = (np.concatenate(pix) if pix else np.zeros(0, np.int64)).astype(np.int32)
        self.ent_blk = np.repeat(np.arange(self.K, dtype=np.int32), self.sizes)
        self.mem_ent = np.argsort(self.ent_pix, kind="stable").astype(np.int64)   # blocks ascending
        cnt = np.bincount(self.ent_pix, minlength=self.n)
        self.mem_ptr = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(cnt, out=self.mem_ptr[1:])
        self.q = cnt.astype(np.float64)
        if self.n and cnt.min() < 1:
            raise ValueError("the partition leaves pixels uncovered")
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=device)
        self.d_blk_ptr, self.d_ent_pix, self.d_ent_blk = t(self.blk_ptr), t(self.ent_pix), t(self.ent_blk)
        self.d_mem_ptr, self.d_mem_ent, self.d_q = t(self.mem_ptr), t(self.mem_ent), t(self.q)

    def fill(self, G: _lib.GStep) -> _lib.GStep:
        G.n, G.K, G.M = self.n, self.K, self.M
        G.blk_ptr, G.ent_pix, G.ent_blk = (self.d_blk_ptr.data_ptr(), self.d_ent_pix.data_ptr(),
                                          self.d_ent_blk.data_ptr())
        G.mem_ptr, G.mem_ent, G.q = (self.d_mem_ptr.data_ptr(), self.d_mem_ent.data_ptr(),
                                     self.d_q.data_ptr())
        return G

    def desc(self) -> _lib.GStep:
        return self.fill(_lib.GStep())

    # host <-> entry-indexed vectors
    def split(self, cat: np.ndarray) -> list:
        return [cat[self.blk_ptr[k]:self.blk_ptr[k + 1]] for k in range(self.K)]

    def join(self, per_block, dtype, what: str) -> np.ndarray:
        if len(per_block) != self.K:
            raise ValueError(f"expected {self.K} block {what}, got {len(per_block)}")
        out = np.empty(self.M, dtype=dtype)
        for k, v in enumerate(per_block):
            v = np.asarray(v)
            if v.shape != (int(self.sizes[k]),):
                raise ValueError(f"block {k} {what} has shape {v.shape}, expected ({self.sizes[k]},)")
            out[self.blk_ptr[k]:self.blk_ptr[k + 1]] = v
        return out


def layout(partition: Partition) -> PartitionLayout:
    return _cached(_layouts, partition, lambda: PartitionLayout(partition, _device()))


class ModelArrays:
    """Device copies of a model: the unary and the canonical pair list (eager),
    the symmetric CSR of W with duplicate pairs summed, like SparseWeights.to_csr
    (on first use: the step kernels need it, evaluate_energy does not)."""

    def __init__(self, model: EnergyModel, device):
        import torch
        self.model, self.device = model, device
        w = model.weights
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=device)
        self.u = t(model.unary)
        self.pi, self.pj, self.pw = t(w.rows.astype(np.int32)), t(w.cols.astype(np.int32)), t(w.vals)
        self.npairs = int(w.npairs)
        self.energy_scratch = torch.zeros(int(_lib.lib().dope_gs_energy_scratch()) + 3,
                                          dtype=torch.float64, device=device)
        self._csr = False

    def csr(self) -> "ModelArrays":
        if self._csr:
            return self
        import torch
        w = self.model.weights
        n = w.n
        src = np.concatenate([w.rows, w.cols]).astype(np.int64)
        dst = np.concatenate([w.cols, w.rows]).astype(np.int64)
        val = np.concatenate([w.vals, w.vals])
        order = np.lexsort((dst, src))
        src, dst, val = src[order], dst[order], val[order]
        if src.size:
            first = np.ones(src.size, dtype=bool)
            first[1:] = (src[1:] != src[:-1]) | (dst[1:] != dst[:-1])
            starts = np.flatnonzero(first)
            val = np.add.reduceat(val, starts)
            src, dst = src[starts], dst[starts]
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(src, minlength=n), out=ptr[1:])
        deg = np.zeros(n)
        np.add.at(deg, src, val)
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=self.device)
        self.adj_ptr_h, self.adj_idx_h, self.adj_w_h, self.deg_h = ptr, dst.astype(np.int32), val, deg
        self.adj_ptr, self.adj_idx, self.adj_w, self.deg = t(ptr), t(dst.astype(np.int32)), t(val), t(deg)
        self._csr = True
        return self


def model_arrays(model: EnergyModel) -> ModelArrays:
    return _cached(_models, model, lambda: ModelArrays(model, _device()))


def device_energy(model: EnergyModel, y) -> float:
    """evaluate_energy (energy.py:187-194) on the device, deterministic order."""
    import torch
    dev = _device()
    ma = model_arrays(model)
    yt = y if isinstance(y, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(y, dtype=np.float64),
                                                              device=dev)
    yt = yt.to(device=dev, dtype=torch.float64).contiguous()
    if tuple(yt.shape) != (model.n,):
        raise ValueError(f"labeling has shape {tuple(yt.shape)}, expected ({model.n},)")
    nsc = int(_lib.lib().dope_gs_energy_scratch())
    out = ma.energy_scratch[nsc:]
    _lib.check(_lib.lib().dope_gs_energy(model.n, ma.u.data_ptr(), ma.npairs,
                                         ma.pi.data_ptr() if ma.npairs else None,
                                         ma.pj.data_ptr() if ma.npairs else None,
                                         ma.pw.data_ptr() if ma.npairs else None, float(model.lam),
                                         yt.data_ptr(), ma.energy_scratch.data_ptr(), out.data_ptr(),
                                         _stream(dev)), "dope_gs_energy")
    return float(out[0].item())


class BlockView:
    """One block's BlockProblem fields (blockform.py:32-45), materialised on the
    host on demand (the device kernels never need them)."""

    def __init__(self, problems: "GraphProblems", k: int):
        self._p, self.k = problems, k
        self.block = problems.partition.blocks[k]

    @property
    def size(self) -> int:
        return int(self._p.layout.sizes[self.k])

    @property
    def pixels(self) -> np.ndarray:
        lay = self._p.layout
        return lay.ent_pix[lay.blk_ptr[self.k]:lay.blk_ptr[self.k + 1]].astype(np.int64)

    @property
    def u_hat(self) -> np.ndarray:
        p = self.pixels
        return self._p.model.unary[p] * (1.0 / self._p.layout.q[p])

    @property
    def w_hat(self):
        from .energy import SparseWeights
        g = self._p
        a, b = g.bp_ptr[self.k], g.bp_ptr[self.k + 1]
        return SparseWeights(self.size, g.bp_i[a:b], g.bp_j[a:b], g.bp_w[a:b], allow_negative=True)

    @property
    def d_hat(self) -> np.ndarray:
        return self.w_hat.degrees()

    @property
    def r_diag(self) -> np.ndarray:
        lay = self._p.layout
        return self._p.r[lay.blk_ptr[self.k]:lay.blk_ptr[self.k + 1]].cpu().numpy()

    @property
    def c_rows(self):
        """Coupling rows C[i, j] = (L[g, j] / q_g) * m_j as scipy CSR (block rows x n)."""
        import scipy.sparse as sp
        g = self._p
        lay, ma = g.layout, g.arrays
        p = self.pixels
        inblk = np.zeros(lay.n, dtype=bool)
        inblk[p] = True
        rows, cols, vals = [], [], []
        for i, gp in enumerate(p):
            qi = 1.0 / lay.q[gp]
            a, b = ma.adj_ptr_h[gp], ma.adj_ptr_h[gp + 1]
            js = ma.adj_idx_h[a:b].astype(np.int64)
            m = np.where(inblk[js], 1.0 - 1.0 / lay.q[js], 1.0)
            rows.append(np.full(js.size + 1, i))
            cols.append(np.concatenate([js, [gp]]))
            vals.append(np.concatenate([(qi * -ma.adj_w_h[a:b]) * m, [(qi * ma.deg_h[gp]) * (1.0 - qi)]]))
        mat = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                            shape=(self.size, lay.n))
        mat.eliminate_zeros()
        return mat


class GraphProblems:
    """assemble_block_problems (blockform.py:48-86) on the device for any model
    and partition: the partition layout, the model's CSR, the remainders r and
    every block's in-block pairs with rescaled weights w / (q_i q_j)."""

    def __init__(self, model: EnergyModel, partition: Partition):
        import torch
        if model.n != partition.shape.n:
            raise ValueError("model and partition sizes differ")
        self.model, self.partition = model, partition
        dev = self.device = _device()
        self.layout = layout(partition)
        self.arrays = model_arrays(model).csr()
        lay, ma = self.layout, self.arrays
        self.r = torch.zeros(max(lay.M, 1), dtype=torch.float64, device=dev)
        G = self.desc()
        _lib.check(_lib.lib().dope_gs_prepare(C.byref(G), self.r.data_ptr(), _stream(dev)), "dope_gs_prepare")
        self._block_pairs()

    def desc(self) -> _lib.GStep:
        G = self.layout.desc()
        ma = self.arrays
        G.adj_ptr, G.adj_idx, G.adj_w = ma.adj_ptr.data_ptr(), ma.adj_idx.data_ptr(), ma.adj_w.data_ptr()
        G.deg, G.u, G.r = ma.deg.data_ptr(), ma.u.data_ptr(), self.r.data_ptr()
        return G

    def _block_pairs(self):
        """In-block pairs (block-local i < j, row-major like w_scaled[p][:, p]) and
        their weights (w_ij / q_i) / q_j."""
        import torch
        lay, w = self.layout, self.model.weights
        qmax = int(lay.q.max()) if lay.n else 1
        gi, gj, gw = w.rows.astype(np.int64), w.cols.astype(np.int64), w.vals
        blocks, li, lj, vals = [], [], [], []
        for s in range(qmax):   # the s-th block holding pixel i ...
            has = lay.mem_ptr[gi] + s < lay.mem_ptr[gi + 1]
            ei = lay.mem_ent[lay.mem_ptr[gi[has]] + s]
            kb = lay.ent_blk[ei]
            pj_ = gj[has]
            for t in range(qmax):   # ... is also the t-th block holding j
                hj = lay.mem_ptr[pj_] + t < lay.mem_ptr[pj_ + 1]
                ej = np.full(pj_.size, -1, dtype=np.int64)
                ej[hj] = lay.mem_ent[lay.mem_ptr[pj_[hj]] + t]
                ok = hj & (lay.ent_blk[np.maximum(ej, 0)] == kb)
                if not ok.any():
                    continue
                a = ei[ok] - lay.blk_ptr[kb[ok]]
                b = ej[ok] - lay.blk_ptr[kb[ok]]
                lo, hi = np.minimum(a, b), np.maximum(a, b)
                qa = lay.q[gi[has][ok]]
                qb = lay.q[pj_[ok]]
                blocks.append(kb[ok].astype(np.int64))
                li.append(lo)
                lj.append(hi)
                vals.append((1.0 / qa * gw[has][ok]) * (1.0 / qb))
        if blocks:
            kb, li, lj, vals = (np.concatenate(blocks), np.concatenate(li), np.concatenate(lj),
                                np.concatenate(vals))
        else:
            kb = li = lj = np.zeros(0, np.int64)
            vals = np.zeros(0)
        order = np.lexsort((lj, li, kb))
        kb, li, lj, vals = kb[order], li[order], lj[order], vals[order]
        self.bp_ptr = np.zeros(lay.K + 1, dtype=np.int64)
        np.cumsum(np.bincount(kb, minlength=lay.K), out=self.bp_ptr[1:])
        self.bp_i, self.bp_j, self.bp_w = li.astype(np.int32), lj.astype(np.int32), vals
        # every block's tail-grouped arc lists in pair order (built once here,
        # not per solve): arc 2p leaves i, arc 2p + 1 leaves j
        m_b = lay.sizes
        P_b = np.diff(self.bp_ptr)
        arc_tail = np.empty(2 * li.size, dtype=np.int64)
        arc_tail[0::2] = li
        arc_tail[1::2] = lj
        arc_blk = np.repeat(kb, 2)
        arc_local = np.arange(2 * li.size, dtype=np.int64) - 2 * np.repeat(self.bp_ptr[:-1], 2 * P_b)
        order = np.lexsort((arc_local, arc_tail, arc_blk))
        adj = arc_local[order].astype(np.int32)
        counts = np.zeros(lay.M + lay.K, dtype=np.int64)   # per block m_b + 1 slots, slot 0 stays 0
        ent_slot = arc_tail + lay.blk_ptr[arc_blk] + arc_blk + 1
        np.add.at(counts, ent_slot, 1)
        adj_off = np.zeros(lay.M + lay.K, dtype=np.int64)
        for b in range(lay.K):   # per-block prefix sums (K small Python steps)
            a0 = int(lay.blk_ptr[b]) + b
            adj_off[a0:a0 + m_b[b] + 1] = np.cumsum(counts[a0:a0 + m_b[b] + 1])
        self.adj_off_h, self.adj_h = adj_off.astype(np.int32), adj
        neg = np.flatnonzero(vals < 0)
        self.first_nonsubmodular = int(kb[neg[0]]) if neg.size else -1
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=self.device)
        self.d_bp_ptr, self.d_bp_i, self.d_bp_j, self.d_bp_w = (t(self.bp_ptr), t(self.bp_i), t(self.bp_j),
                                                                t(vals))
        self.d_adj_off = t(self.adj_off_h)
        self.d_adj = t(self.adj_h) if self.adj_h.size else t(np.zeros(1, np.int32))
        self._ws = None

    def __len__(self) -> int:
        return self.layout.K

    def __getitem__(self, k: int) -> BlockView:
        if not -len(self) <= k < len(self):
            raise IndexError(k)
        return BlockView(self, k % len(self))

    def __iter__(self):
        return (self[k] for k in range(len(self)))

    # -- kernels ----------------------------------------------------------------
    def objective(self, y, a, mu: float, lam: float, entries=None):
        import torch
        if mu < 0 or lam < 0:
            raise ValueError("mu and lambda must be non-negative")   # blockform.py:98-99
        lin = torch.zeros(max(self.layout.M, 1), dtype=torch.float64, device=self.device)
        e0, e1 = entries if entries is not None else (0, self.layout.M)
        G = self.desc()
        _lib.check(_lib.lib().dope_gs_objective(C.byref(G), e0, e1, y.data_ptr(), a.data_ptr(),
                                                float(mu), float(lam), lin.data_ptr(), _stream(self.device)),
                   "dope_gs_objective")
        return lin

    def _workspace(self):
        import torch
        if self._ws is None:
            lb = _lib.lib()
            lay = self.layout
            sizes = [int(lb.dope_bk_workspace_bytes(int(lay.sizes[k]),
                                                    int(self.bp_ptr[k + 1] - self.bp_ptr[k])))
                     for k in range(lay.K)]
            off = np.zeros(lay.K + 1, dtype=np.int64)
            np.cumsum(sizes, out=off[1:])
            self._ws = (torch.empty(max(int(off[-1]), 8), dtype=torch.uint8, device=self.device),
                        torch.as_tensor(off, device=self.device))
        return self._ws

    def solve(self, lin, lam: float, kind: str):
        """Every block's min cut (or exhaustive minimum) -> entry-indexed labels."""
        import torch
        lay = self.layout
        lb = _lib.lib()
        labels = torch.zeros(max(lay.M, 1), dtype=torch.uint8, device=self.device)
        out = torch.zeros(max(lay.K, 1), dtype=torch.float64, device=self.device)
        st = _stream(self.device)
        P = int(self.bp_ptr[-1])
        pp = lambda t: t.data_ptr() if P else None
        if kind == "maxflow":
            if self.first_nonsubmodular >= 0:
                from .admm import BlockSolveError
                raise BlockSolveError(self.first_nonsubmodular, NonSubmodularError(
                    "pairwise weights contain negative entries; max-flow requires a submodular instance"))
            caps = self.d_bp_w * float(lam)
            ws, ws_off = self._workspace()
            _lib.check(lb.dope_bk_maxflow_batch(lay.K, lay.d_blk_ptr.data_ptr(), self.d_bp_ptr.data_ptr(),
                                                ws_off.data_ptr(), lin.data_ptr(), pp(self.d_bp_i), pp(self.d_bp_j),
                                                pp(caps), pp(caps), labels.data_ptr(), out.data_ptr(),
                                                ws.data_ptr(), self.d_adj_off.data_ptr(), self.d_adj.data_ptr(),
                                                st), "dope_bk_maxflow_batch")
        elif kind == "exhaustive":
            big = np.flatnonzero(lay.sizes > EXHAUSTIVE_MAX_VARS)
            if big.size:
                from .admm import BlockSolveError
                raise BlockSolveError(int(big[0]), ValueError(
                    f"exhaustive solver limited to {EXHAUSTIVE_MAX_VARS} variables, got {lay.sizes[big[0]]}"))
            _lib.check(lb.dope_exhaustive_batch(lay.K, lay.d_blk_ptr.data_ptr(), self.d_bp_ptr.data_ptr(),
                                                lin.data_ptr(), pp(self.d_bp_i), pp(self.d_bp_j), pp(self.d_bp_w),
                                                float(lam), labels.data_ptr(), out.data_ptr(), st),
                       "dope_exhaustive_batch")
        else:
            raise NotImplementedError(f"the {kind!r} block solver has no B200 kernel "
                                      "(ICM's sequential sweep order is out of scope)")
        return labels

    def solve_global(self, yhat, a, mu: float, lam: float, clamp: bool):
        import torch
        if not mu > 0:
            raise ValueError("global update requires mu > 0")   # admm.py:143-144
        y = torch.empty(max(self.layout.n, 1), dtype=torch.float64, device=self.device)
        flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        G = self.desc()
        _lib.check(_lib.lib().dope_gs_solve_global(C.byref(G), yhat.data_ptr(), a.data_ptr(), float(mu),
                                                   float(lam), y.data_ptr(), int(clamp), flag.data_ptr(),
                                                   _stream(self.device)), "dope_gs_solve_global")
        return y[:self.layout.n], flag

    def consensus_parts(self, yhat, a, y):
        import torch
        out = torch.zeros(max(2 * self.layout.K, 2), dtype=torch.float64, device=self.device)
        G = self.desc()
        _lib.check(_lib.lib().dope_gs_consensus_objective(C.byref(G), yhat.data_ptr(), a.data_ptr(),
                                                          y.data_ptr(), out.data_ptr(), _stream(self.device)),
                   "dope_gs_consensus_objective")
        return out[:2 * self.layout.K].cpu().numpy().reshape(-1, 2)


def problems_for(model: EnergyModel, partition: Partition) -> GraphProblems:
    return GraphProblems(model, partition)


def residuals_sq(lay: PartitionLayout, yhat, y):
    import torch
    ss = torch.zeros(max(lay.K, 1), dtype=torch.float64, device=lay.device)
    G = lay.desc()
    _lib.check(_lib.lib().dope_gs_residuals(C.byref(G), yhat.data_ptr(), y.data_ptr(), ss.data_ptr(),
                                            _stream(lay.device)), "dope_gs_residuals")
    return ss[:lay.K]


def update_multipliers_dev(lay: PartitionLayout, yhat, y, a):
    G = lay.desc()
    _lib.check(_lib.lib().dope_gs_update_multipliers(C.byref(G), yhat.data_ptr(), y.data_ptr(), a.data_ptr(),
                                                     _stream(lay.device)), "dope_gs_update_multipliers")


def run_graph(model: EnergyModel, partition: Partition, config, problems: GraphProblems | None = None):
    """admm.run (admm.py:207-252) on the general graph path: device compute,
    host bookkeeping of four scalars per iteration."""
    import time

    import torch
    from .admm import AdmmState, TraceRecord, binarize
    gp = problems if isinstance(problems, GraphProblems) else GraphProblems(model, partition)
    lay = gp.layout
    dev = gp.device
    mu0 = config.resolved_mu0(partition.shape.ndim)
    eps = config.resolved_eps(partition)
    lam = float(model.lam)
    y = torch.full((max(lay.n, 1),), 0.5, dtype=torch.float64, device=dev)[:lay.n]
    a = torch.zeros(max(lay.M, 1), dtype=torch.float64, device=dev)
    yhat = torch.zeros(max(lay.M, 1), dtype=torch.uint8, device=dev)
    best_y = y.clone()
    best_e = math.inf
    mu = float(mu0)
    trace, best_it, converged, it = [], 0, False, 0
    for it in range(1, config.max_iters + 1):
        t0 = time.perf_counter()
        mu_at_solve = mu
        lin = gp.objective(y, a, mu, lam)
        yhat = gp.solve(lin, lam, config.solver.kind)
        y, flag = gp.solve_global(yhat, a, mu, lam, clamp=True)
        ss = residuals_sq(lay, yhat, y)
        energy = device_energy(model, y)
        res = np.sqrt(ss.cpu().numpy())
        torch.cuda.current_stream(dev).synchronize()
        trace.append(TraceRecord(it, mu_at_solve, energy, float(np.dot(res, res)),
                                 float(res.max()) if res.size else 0.0, (time.perf_counter() - t0) * 1e3,
                                 bool(flag.item())))
        if energy < best_e:
            best_e, best_it = energy, it
            best_y = y.clone()
        update_multipliers_dev(lay, yhat, y, a)
        mu *= config.mu_fact
        if res.size == 0 or res.max() <= eps:
            converged = True
            break
    if not converged:
        y = best_y
    state = AdmmState.from_device(partition, y=y, yhat_cat=yhat, a_cat=a, layout=lay, mu=mu)
    state.iteration, state.converged, state.best_iteration = it, converged, best_it
    state.trace = trace
    state.clamped_last = trace[-1].clamped if trace else False
    return binarize(state.y), state
