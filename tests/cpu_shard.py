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
