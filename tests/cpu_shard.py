"""CPU shard executor for the multi-process protocol tests (TEST INFRASTRUCTURE).

Implements the shard interface of paper_1704_03116_b200/sharded.py
(run_shards) with numpy and the oracle's BK (the reference's max-flow
restated), so the sharded protocol and DistComm run over gloo on CPU.  It
follows the kernels' per-shard semantics: a slab of whole blocks along axis 0
with one ghost row / plane on each side; the block objective reads the
neighbour rows from the ghost rows; the consensus pass fills this shard's
slot of the agg table [energy of the previous iterate, sum ss, sum of
rounding excesses, max ss, clamp, end-of-run energy] with exact integers; the
ghost rows' new iterate and multipliers are recomputed locally
(dope_ghost_consensus) instead of exchanged; decide() reduces the gathered
table in shard order.  2D and 3D lattices.
"""
import numpy as np
import torch

import oracle as orc

AGG_SLOT = 8


def rsq_excess(ss: np.ndarray) -> np.ndarray:
    """(fl(fl(sqrt(ss))^2) - ss) * 2^53, exact (dope_lattice.cu rsq_excess)."""
    ss = ss.astype(np.float64)
    r = np.sqrt(ss)
    return ((r * r - ss) * 9007199254740992.0).astype(np.int64)


class CpuShardND:
    def __init__(self, u, dims, kpa, lamw, mu, max_iters, kb0, kb1, index=0, count=1):
        dims, kpa = tuple(dims), tuple(kpa)
        self.nd = len(dims)
        self.bs = tuple(d // k for d, k in zip(dims, kpa))
        self.kpa = kpa
        self.kb0, self.kb1 = kb0, kb1
        self.r0, self.r1 = kb0 * self.bs[0], kb1 * self.bs[0]
        self.ldims = (self.r1 - self.r0,) + dims[1:]
        self.u = u.reshape(dims)[self.r0:self.r1].astype(np.int64)
        self.lamw, self.mu, self.q = lamw, mu, lamw // mu
        self.gup, self.gdn = kb0 > 0, kb1 < kpa[0]
        self.max_iters = max_iters
        self.index, self.count = index, count
        self.unit = int(np.prod(dims[1:]))
        self.agg = torch.zeros(AGG_SLOT * count, dtype=torch.int64)
        self.halo = torch.zeros(4 * self.unit, dtype=torch.uint8)
        # block-internal pairs (forward neighbours along every axis), block-local indices
        idx = np.arange(int(np.prod(self.bs))).reshape(self.bs)
        pi, pj = [], []
        for ax in range(self.nd):
            lo = [slice(None)] * self.nd
            hi = [slice(None)] * self.nd
            lo[ax], hi[ax] = slice(0, -1), slice(1, None)
            pi.append(idx[tuple(lo)].ravel())
            pj.append(idx[tuple(hi)].ravel())
        self.pi = np.concatenate(pi).astype(np.int32)
        self.pj = np.concatenate(pj).astype(np.int32)

    def init(self):
        shp = (self.ldims[0] + 2,) + self.ldims[1:]
        self.y2 = np.ones(shp, dtype=np.int64)
        self.yh = np.zeros(shp, dtype=np.int64)
        self.a = np.zeros(self.ldims, dtype=np.int64)
        self.ga = np.zeros((2,) + self.ldims[1:], dtype=np.int64)   # ghost multipliers (up, down)
        self.y2_prev = None
        self.best_e, self.best_it, self.best_y2 = None, 0, self.y2[1:-1].copy()
        self.it, self.converged, self.stop = 0, False, False
        self.trace_e, self.trace_mr, self.trace_rs, self.trace_cl = [], [], [], []

    def _cross_axes(self, loc, first_axis):
        """sum over cross-block neighbours j along the in-slab axes of (loc_v - loc_j);
        loc is the slab (first_axis 1) or one ghost layer (first_axis 0)."""
        s = np.zeros(loc.shape, dtype=np.int64)
        for ax in range(first_axis, loc.ndim):
            n, b = loc.shape[ax], self.bs[ax + 1 - first_axis]
            c = np.arange(n)
            shape = [1] * loc.ndim
            shape[ax] = n
            low = ((c % b == 0) & (c > 0)).reshape(shape)
            high = ((c % b == b - 1) & (c < n - 1)).reshape(shape)
            s += np.where(low, loc - np.roll(loc, 1, axis=ax), 0)
            s += np.where(high, loc - np.roll(loc, -1, axis=ax), 0)
        return s

    def _cross(self, arr):
        """sum over cross-block neighbours j of (arr_v - arr_j) for every local voxel
        (arr carries the ghost layers along axis 0)."""
        loc = arr[1:-1]
        s = self._cross_axes(loc, 1)
        n, b = self.ldims[0], self.bs[0]
        c = np.arange(n)
        shape = [n] + [1] * (self.nd - 1)
        low = (c % b == 0)
        low[0] = low[0] and self.gup
        high = (c % b == b - 1)
        high[-1] = high[-1] and self.gdn
        s += np.where(low.reshape(shape), loc - arr[:-2], 0)
        s += np.where(high.reshape(shape), loc - arr[2:], 0)
        return s

    def _blocks(self):
        nb = [self.ldims[a] // self.bs[a] for a in range(self.nd)]
        for k in np.ndindex(*nb):
            yield tuple(slice(k[a] * self.bs[a], (k[a] + 1) * self.bs[a]) for a in range(self.nd))

    def update_blocks(self):
        if self.stop:
            return
        s = self._cross(self.y2)
        lin = (2 * self.u + self.lamw * s + self.mu * (2 * self.a - self.y2[1:-1]) + self.mu) / 2.0
        cap = np.full(self.pi.size, float(self.lamw))
        for sl in self._blocks():
            labels, _ = orc.bk_maxflow(lin[sl].ravel().astype(np.float64), self.pi, self.pj, cap, cap)
            gl = (slice(sl[0].start + 1, sl[0].stop + 1),) + sl[1:]
            self.yh[gl] = labels.reshape(self.bs)

    # -- label halo -----------------------------------------------------------
    def halo_slots(self):
        U = self.unit
        return tuple(self.halo[i * U:(i + 1) * U] for i in range(4))

    def pack_rows(self):
        first, last, _, _ = self.halo_slots()
        first.copy_(torch.from_numpy(self.yh[1].ravel().astype(np.uint8)))
        last.copy_(torch.from_numpy(self.yh[self.ldims[0]].ravel().astype(np.uint8)))

    def install_rows(self):
        _, _, up, dn = self.halo_slots()
        if self.gup:
            self.yh[0] = up.numpy().reshape(self.ldims[1:])
        if self.gdn:
            self.yh[self.ldims[0] + 1] = dn.numpy().reshape(self.ldims[1:])

    def _pair_energy(self, yo):
        e = 0
        for ax in range(1, self.nd):
            e += int(np.abs(np.diff(yo[1:-1], axis=ax)).sum())
        last = self.ldims[0] + 1 if self.gdn else self.ldims[0]
        e += int(np.abs(yo[2:last + 1] - yo[1:last]).sum())
        return self.lamw * e

    def _slot(self):
        return self.agg[AGG_SLOT * self.index:AGG_SLOT * (self.index + 1)]

    def update_global(self):
        if self.stop:
            return
        ypre = self.yh[1:-1] + self.a - self.q * self._cross(self.yh)
        clamped = int(np.any((ypre < 0) | (ypre > 1)))
        y_new = np.clip(ypre, 0, 1)
        yh = self.yh[1:-1]
        ss_blocks = np.array([int(((yh[sl] - y_new[sl]) ** 2).sum()) for sl in self._blocks()])
        e = 0
        if self.it >= 1:
            yo = self.y2 >> 1
            e = int((self.u * yo[1:-1]).sum()) + self._pair_energy(yo)
        slot = self._slot()
        slot[0] = e
        slot[1] = int(ss_blocks.sum())
        slot[2] = int(rsq_excess(ss_blocks).sum())
        slot[3] = int(ss_blocks.max())
        slot[4] = clamped
        self.a = self.a + yh - y_new
        self.y2_prev = self.y2.copy()
        self.y2[1:-1] = 2 * y_new

    def ghost_consensus(self):
        """The ghost layers' new iterate and multipliers from the labels (the owner's update)."""
        if self.stop:
            return
        n = self.ldims[0]
        for side, has, g, inner in ((0, self.gup, 0, 1), (1, self.gdn, n + 1, n)):
            if not has:
                continue
            yg = self.yh[g]
            s = (yg - self.yh[inner]) + self._cross_axes(yg, 0)
            ypre = yg + self.ga[side] - self.q * s
            y = np.clip(ypre, 0, 1)
            self.ga[side] = self.ga[side] + yg - y
            self.y2[g] = 2 * y

    def decide(self):
        if self.stop:
            return
        t = self.agg.view(self.count, AGG_SLOT).numpy()
        E, S, X, M2, F = int(t[:, 0].sum()), int(t[:, 1].sum()), int(t[:, 2].sum()), \
            int(t[:, 3].max()), int(t[:, 4].max())
        R2 = float(S) + float(X) * 2.0 ** -53
        it = self.it
        if it >= 1:
            self.trace_e.append(E)
            if self.best_e is None or E < self.best_e:
                self.best_e, self.best_it = E, it
                self.best_y2 = self.y2_prev[1:-1].copy()
        mr = float(np.sqrt(M2))
        self.trace_rs.append(R2)
        self.trace_mr.append(mr)
        self.trace_cl.append(bool(F))
        self.it = it + 1
        if mr <= 0.0:
            self.converged = self.stop = True

    def energy_local(self):
        yo = self.y2 >> 1
        self._slot()[5] = int((self.u * yo[1:-1]).sum()) + self._pair_energy(yo)

    def finish_decide(self):
        E = int(self.agg.view(self.count, AGG_SLOT)[:, 5].sum())
        self.trace_e.append(E)
        if self.best_e is None or E < self.best_e:
            self.best_e, self.best_it = E, self.it
            self.best_y2 = self.y2[1:-1].copy()
        self.final_y2 = self.y2[1:-1].copy() if self.converged else self.best_y2

    def labels(self):
        return (self.final_y2 >= 1).astype(np.int8)
