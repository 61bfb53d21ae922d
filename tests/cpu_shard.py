"""CPU shard executor for the multi-process protocol tests (TEST INFRASTRUCTURE).

Implements the GpuShard interface of paper_1704_03116_b200/sharded.py with
numpy and the oracle's BK (the reference's max-flow restated), so the sharded
driver and DistComm can be exercised over gloo on CPU.  It follows the same
per-shard semantics as the kernels: the block objective reads the neighbour
rows from ghost rows, the consensus pass publishes local aggregates
[energy of the previous iterate, sum res^2, max res^2, clamp], and decide()
applies the global ones.
"""
import numpy as np
import torch

import oracle as orc


class CpuShard:
    def __init__(self, u, dims, kpa, lamw, mu, max_iters, kb0, kb1):
        H, W = dims
        ky, kx = kpa
        bh, bw = H // ky, W // kx
        self.W, self.bh, self.bw, self.kx = W, bh, bw, kx
        self.kb0, self.kb1, self.ky = kb0, kb1, ky
        self.r0, self.r1 = kb0 * bh, kb1 * bh
        self.Hl = self.r1 - self.r0
        self.u = u.reshape(H, W)[self.r0:self.r1].astype(np.int64)
        self.lamw, self.mu = lamw, mu
        self.q = lamw // mu
        self.gup, self.gdn = kb0 > 0, kb1 < ky
        self.max_iters = max_iters
        self.agg = torch.zeros(4, dtype=torch.int64)
        self.energy_acc = torch.zeros(1, dtype=torch.int64)
        self.rows_i32 = [torch.zeros(W, dtype=torch.int32) for _ in range(4)]
        self.rows_u8 = [torch.zeros(W, dtype=torch.uint8) for _ in range(4)]

    # state: y2 / yhat with a ghost row above (index 0) and below (index Hl+1)
    def init(self):
        self.y2 = np.ones((self.Hl + 2, self.W), dtype=np.int64)
        self.yh = np.zeros((self.Hl + 2, self.W), dtype=np.int64)
        self.a = np.zeros((self.Hl, self.W), dtype=np.int64)
        self.y2_prev = None
        self.best_e, self.best_it, self.best_y2 = None, 0, self.y2[1:-1].copy()
        self.it, self.converged, self.stop = 0, False, False
        self.trace_e, self.trace_mr, self.trace_rs, self.trace_cl = [], [], [], []

    def _cross(self, arr, r, c, lo_r, lo_c):
        """sum over cross-block neighbours of (arr_g - arr_j) for local pixel (r, c)."""
        s = 0
        g = arr[r + 1, c]
        if c == lo_c and c > 0:
            s += g - arr[r + 1, c - 1]
        if c == lo_c + self.bw - 1 and c + 1 < self.W:
            s += g - arr[r + 1, c + 1]
        if r == lo_r and (r > 0 or self.gup):
            s += g - arr[r, c]
        if r == lo_r + self.bh - 1 and (r + 1 < self.Hl or self.gdn):
            s += g - arr[r + 2, c]
        return s

    def update_blocks(self):
        if self.stop:
            return
        bh, bw = self.bh, self.bw
        idx = np.arange(bh * bw).reshape(bh, bw)
        pi = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()]).astype(np.int32)
        pj = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()]).astype(np.int32)
        cap = np.full(pi.size, float(self.lamw))
        for by in range(self.kb1 - self.kb0):
            for bx in range(self.kx):
                lo_r, lo_c = by * bh, bx * bw
                lin = np.empty(bh * bw)
                for rr in range(bh):
                    for cc in range(bw):
                        r, c = lo_r + rr, lo_c + cc
                        s = self._cross(self.y2, r, c, lo_r, lo_c)   # in units of 2y
                        y2g = self.y2[r + 1, c]
                        lin[rr * bw + cc] = (2 * self.u[r, c] + self.lamw * s
                                             + self.mu * (2 * self.a[r, c] - y2g) + self.mu) / 2.0
                labels, _ = orc.bk_maxflow(lin, pi, pj, cap, cap)
                self.yh[1 + lo_r:1 + lo_r + bh, lo_c:lo_c + bw] = labels.reshape(bh, bw)

    def staging(self, which):
        return self.rows_u8 if which == 0 else self.rows_i32

    def pack_rows(self, which):
        first, last, _, _ = self.staging(which)
        src = self.yh if which == 0 else self.y2
        first.copy_(torch.from_numpy(src[1].astype(first.numpy().dtype)))
        last.copy_(torch.from_numpy(src[self.Hl].astype(last.numpy().dtype)))
        return first, last

    def ghost_update(self, which, up, dn):
        dst = self.yh if which == 0 else self.y2
        if up is not None and self.gup:
            dst[0] = up.numpy()
        if dn is not None and self.gdn:
            dst[self.Hl + 1] = dn.numpy()

    def update_global(self):
        if self.stop:
            return
        Hl, W = self.Hl, self.W
        y_new = np.zeros((Hl, W), dtype=np.int64)
        clamped = 0
        for r in range(Hl):
            for c in range(W):
                lo_r, lo_c = (r // self.bh) * self.bh, (c // self.bw) * self.bw
                s = self._cross(self.yh, r, c, lo_r, lo_c)
                ypre = self.yh[r + 1, c] + self.a[r, c] - self.q * s
                clamped |= int(ypre < 0 or ypre > 1)
                y_new[r, c] = min(max(ypre, 0), 1)
        yh = self.yh[1:-1]
        ss_blocks = ((yh - y_new) ** 2).reshape(Hl // self.bh, self.bh, W // self.bw,
                                                self.bw).sum(axis=(1, 3))
        # energy of the previous iterate (pairs (v,right), (v,down) incl. the ghost below)
        e = 0
        if self.it >= 1:
            yo = self.y2 >> 1
            e = int((self.u * yo[1:-1]).sum())
            e += self.lamw * int(np.abs(np.diff(yo[1:-1], axis=1)).sum())
            last = Hl + 1 if self.gdn else Hl
            e += self.lamw * int(np.abs(yo[2:last + 1] - yo[1:last]).sum())
        rs = float(np.sum(np.sqrt(ss_blocks.astype(np.float64)) ** 2))
        self.agg[0] = e
        self.agg[1:2].view(torch.float64)[0] = rs
        self.agg[2] = int(ss_blocks.max())
        self.agg[3] = clamped
        self.a = self.a + yh - y_new
        self.y2_prev = self.y2.copy()
        self.y2[1:-1] = 2 * y_new

    def decide(self):
        if self.stop:
            return
        E, M2, F = int(self.agg[0]), int(self.agg[2]), int(self.agg[3])
        R2 = float(self.agg[1:2].view(torch.float64)[0])
        t = self.it
        if t >= 1:
            self.trace_e.append(E)
            if self.best_e is None or E < self.best_e:
                self.best_e, self.best_it = E, t
                self.best_y2 = self.y2_prev[1:-1].copy()
        mr = float(np.sqrt(M2))
        self.trace_rs.append(R2)
        self.trace_mr.append(mr)
        self.trace_cl.append(bool(F))
        self.it = t + 1
        if mr <= 0.0:
            self.converged = self.stop = True

    def energy_local(self):
        yo = self.y2 >> 1
        Hl = self.Hl
        e = int((self.u * yo[1:-1]).sum()) + self.lamw * int(np.abs(np.diff(yo[1:-1], axis=1)).sum())
        last = Hl + 1 if self.gdn else Hl
        e += self.lamw * int(np.abs(yo[2:last + 1] - yo[1:last]).sum())
        self.energy_acc[0] = e

    def finish_decide(self):
        E = int(self.energy_acc[0])
        self.trace_e.append(E)
        if self.best_e is None or E < self.best_e:
            self.best_e, self.best_it = E, self.it
            self.best_y2 = self.y2[1:-1].copy()
        self.final_y2 = self.y2[1:-1].copy() if self.converged else self.best_y2

    def labels(self):
        return (self.final_y2 >= 1).astype(np.int8)


class CpuShardND:
    """GpuShard interface for 2D and 3D lattices (slab of whole blocks along
    axis 0 with one ghost row / plane on each side), vectorised numpy + the
    oracle's BK per block.  Same per-shard semantics as the kernels."""

    def __init__(self, u, dims, kpa, lamw, mu, max_iters, kb0, kb1):
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
        self.W = int(np.prod(dims[1:]))
        self.agg = torch.zeros(4, dtype=torch.int64)
        self.energy_acc = torch.zeros(1, dtype=torch.int64)
        self.rows_u8 = [torch.zeros(self.W, dtype=torch.uint8) for _ in range(4)]
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
        self.y2_prev = None
        self.best_e, self.best_it, self.best_y2 = None, 0, self.y2[1:-1].copy()
        self.it, self.converged, self.stop = 0, False, False
        self.trace_e, self.trace_mr, self.trace_rs, self.trace_cl = [], [], [], []

    def _cross(self, arr):
        """sum over cross-block neighbours j of (arr_v - arr_j) for every local voxel
        (arr carries the ghost layers along axis 0)."""
        loc = arr[1:-1]
        s = np.zeros(self.ldims, dtype=np.int64)
        for ax in range(self.nd):
            n, b = self.ldims[ax], self.bs[ax]
            c = np.arange(n)
            shape = [1] * self.nd
            shape[ax] = n
            low = (c % b == 0).reshape(shape)
            high = (c % b == b - 1).reshape(shape)
            if ax == 0:
                prev, nxt = arr[:-2], arr[2:]
                has_prev = np.ones(n, bool)
                has_prev[0] = self.gup
                has_next = np.ones(n, bool)
                has_next[-1] = self.gdn
            else:
                prev = np.roll(loc, 1, axis=ax)
                nxt = np.roll(loc, -1, axis=ax)
                has_prev = c > 0
                has_next = c < n - 1
            s += np.where(low & has_prev.reshape(shape), loc - prev, 0)
            s += np.where(high & has_next.reshape(shape), loc - nxt, 0)
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

    def staging(self, which):
        return self.rows_u8

    def pack_rows(self, which):
        first, last, _, _ = self.staging(which)
        src = self.yh if which == 0 else self.y2
        first.copy_(torch.from_numpy(src[1].ravel().astype(np.uint8)))
        last.copy_(torch.from_numpy(src[self.ldims[0]].ravel().astype(np.uint8)))
        return first, last

    def ghost_update(self, which, up, dn):
        dst = self.yh if which == 0 else self.y2
        if up is not None and self.gup:
            dst[0] = up.numpy().reshape(self.ldims[1:])
        if dn is not None and self.gdn:
            dst[self.ldims[0] + 1] = dn.numpy().reshape(self.ldims[1:])

    def _pair_energy(self, yo):
        e = 0
        for ax in range(1, self.nd):
            e += int(np.abs(np.diff(yo[1:-1], axis=ax)).sum())
        last = self.ldims[0] + 1 if self.gdn else self.ldims[0]
        e += int(np.abs(yo[2:last + 1] - yo[1:last]).sum())
        return self.lamw * e

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
        rs = float(np.sum(np.sqrt(ss_blocks.astype(np.float64)) ** 2))
        self.agg[0] = e
        self.agg[1:2].view(torch.float64)[0] = rs
        self.agg[2] = int(ss_blocks.max())
        self.agg[3] = clamped
        self.a = self.a + yh - y_new
        self.y2_prev = self.y2.copy()
        self.y2[1:-1] = 2 * y_new

    decide = CpuShard.decide
    finish_decide = CpuShard.finish_decide
    labels = CpuShard.labels

    def energy_local(self):
        yo = self.y2 >> 1
        self.energy_acc[0] = int((self.u * yo[1:-1]).sum()) + self._pair_energy(yo)
