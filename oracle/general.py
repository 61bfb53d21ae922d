"""CPU oracle of the general path (TEST INFRASTRUCTURE ONLY).

Restates, for a 2D 4/8-connected lattice model, the reference's loop on an
overlapping box partition with an arbitrary mu schedule:

  partition      partition.py:62-108 (axis ranges grown by
                 ceil(pct/100 * len / 2), block counts q)
  block problem  blockform.py:48-86 (u/q, w/(q_i q_j), r = d/q^2 - dhat,
                 c_rows = rows of diag(1/q)(D - W) masked by (1 - 1/q_j) on
                 in-block columns) and block_objective (blockform.py:89-105)
  block solve    solvers.solve_block -> maxflow.build_graph / min_cut
                 (maxflow.py:73-113) via the oracle's BK restatement
  global step    solve_global + clamp (admm.py:136-180)
  residuals      block_residuals (admm.py:193-199)
  energy         evaluate_energy (energy.py:187-194)
  loop           admm.run (admm.py:207-252): trace, strict-< best, mu *= fact,
                 stop when max residual <= eps, best iterate on exit

The stencil form replaces the reference's sparse matrices; float operation
order differs (results agree within the float parity bar).  Pinned against
the reference's own fixtures (tests/golden/gen_*.npz) by
tests/test_oracle_general.py.  Only tests/ and bench.py's CPU-baseline leg
import this module.
"""
from __future__ import annotations

import math

import numpy as np

import oracle as orc

# neighbour offsets (dy, dx) of the 8-connected stencil; forward = first four
DIRS = [(0, 1), (1, 0), (1, 1), (1, -1), (0, -1), (-1, 0), (-1, -1), (-1, 1)]


def axis_ranges(dim: int, k: int, overlap_pct: int) -> list:
    base, rem = divmod(dim, k)
    out, lo = [], 0
    for r in range(k):
        length = base + (1 if r < rem else 0)
        hi = lo + length
        grow = math.ceil(overlap_pct / 100.0 * length / 2.0)
        out.append((max(0, lo - grow), min(dim, hi + grow)))
        lo = hi
    return out


class GeneralSpec:
    """Lattice model: u [H*W], forward weight planes E S SE SW (pair stored at
    its lower pixel), connectivity, lambda; box partition kpa + overlap."""

    def __init__(self, dims, conn, u, planes, lam, kpa, overlap_pct):
        self.H, self.W = dims
        self.conn = conn
        self.u = np.asarray(u, dtype=np.float64).reshape(self.H, self.W)
        self.fw = [np.asarray(p, dtype=np.float64).reshape(self.H, self.W) for p in planes]
        self.lam = float(lam)
        ry = axis_ranges(self.H, kpa[0], overlap_pct)
        rx = axis_ranges(self.W, kpa[1], overlap_pct)
        self.boxes = [(r, c) for r in ry for c in rx]
        q = np.zeros((self.H, self.W), dtype=np.int64)
        for (r0, r1), (c0, c1) in self.boxes:
            q[r0:r1, c0:c1] += 1
        self.q = q.astype(np.float64)
        nd = 8 if conn == 8 else 4
        self.dirs = [d for d in DIRS if conn == 8 or (abs(d[0]) + abs(d[1]) == 1)][:nd]
        # full neighbour weight planes per direction (0 outside the grid)
        self.wd = [self._wplane(dy, dx) for dy, dx in self.dirs]
        self.deg = sum(self.wd)

    def _wplane(self, dy, dx):
        H, W = self.H, self.W
        fwd = {(0, 1): 0, (1, 0): 1, (1, 1): 2, (1, -1): 3}
        out = np.zeros((H, W))
        if (dy, dx) in fwd:
            p = self.fw[fwd[(dy, dx)]]
            out[max(0, -dy):H - max(0, dy), max(0, -dx):W - max(0, dx)] = \
                p[max(0, -dy):H - max(0, dy), max(0, -dx):W - max(0, dx)]
            return out
        # backward: w(p, p + off) = forward plane at p + off
        p = self.fw[fwd[(-dy, -dx)]]
        ys, xs = slice(max(0, -dy), H - max(0, dy)), slice(max(0, -dx), W - max(0, dx))
        yt, xt = slice(max(0, -dy) + dy, H - max(0, dy) + dy), slice(max(0, -dx) + dx, W - max(0, dx) + dx)
        out[ys, xs] = p[yt, xt]
        return out

    def shift(self, a, dy, dx, fill=0.0):
        """out[y, x] = a[y + dy, x + dx] (fill outside)."""
        H, W = a.shape
        out = np.full_like(a, fill)
        out[max(0, -dy):H - max(0, dy), max(0, -dx):W - max(0, dx)] = \
            a[max(0, dy):H - max(0, -dy), max(0, dx):W - max(0, -dx)]
        return out


class _Block:
    """Block k on its window (box plus a one-pixel ring, clipped to the grid):
    every quantity the block touches lives there."""

    def __init__(self, spec: GeneralSpec, k: int):
        (r0, r1), (c0, c1) = spec.boxes[k]
        H, W = spec.H, spec.W
        self.box = (r0, r1, c0, c1)
        self.wr0, self.wr1 = max(0, r0 - 1), min(H, r1 + 1)
        self.wc0, self.wc1 = max(0, c0 - 1), min(W, c1 + 1)
        self.win = (slice(self.wr0, self.wr1), slice(self.wc0, self.wc1))
        self.bl = (slice(r0 - self.wr0, r1 - self.wr0), slice(c0 - self.wc0, c1 - self.wc0))   # box in window
        shp = (self.wr1 - self.wr0, self.wc1 - self.wc0)
        self.inbox = np.zeros(shp, dtype=bool)
        self.inbox[self.bl] = True
        self.q = spec.q[self.win]
        self.deg = spec.deg[self.win]
        self.wd = [w[self.win] for w in spec.wd]
        self.nin, dhat = [], np.zeros(shp)
        for (dy, dx), w in zip(spec.dirs, self.wd):
            nb_in = spec.shift(self.inbox.astype(np.float64), dy, dx) > 0
            nq = spec.shift(self.q, dy, dx, fill=1.0)
            self.nin.append((nb_in, nq))
            dhat += np.where(nb_in & (w != 0), w / (self.q * nq), 0.0)
        self.rdiag = self.deg / (self.q * self.q) - dhat


def run(spec: GeneralSpec, mu0: float, mu_fact: float, eps: float, max_iters: int) -> dict:
    H, W = spec.H, spec.W
    lam = spec.lam
    blocks = [_Block(spec, k) for k in range(len(spec.boxes))]
    nf = 4 if spec.conn == 8 else 2
    y = np.full((H, W), 0.5)
    a = [np.zeros((b.box[1] - b.box[0], b.box[3] - b.box[2])) for b in blocks]
    yh = [np.zeros_like(x, dtype=np.int8) for x in a]
    mu = float(mu0)
    best_e, best_y, best_it = math.inf, y.copy(), 0
    tr = dict(mu=[], energy=[], residual_sq=[], max_block_residual=[], clamped=[])
    converged = False
    it = 0
    for it in range(1, max_iters + 1):
        # ---- block solves (blockform.py:89-105, maxflow.py:73-113) ----
        for k, b in enumerate(blocks):
            q = b.q
            yw = y[b.win]
            cy = (b.deg / q) * (1.0 - 1.0 / q) * yw
            for ((dy, dx), w), (nb_in, nq) in zip(zip(spec.dirs, b.wd), b.nin):
                ny = spec.shift(yw, dy, dx)
                cy += np.where(nb_in, (-w / q) * (1.0 - 1.0 / nq) * ny, (-w / q) * ny)
            lin = spec.u[b.win] / q + lam * (cy + b.rdiag * yw) + mu * ((0.0 - yw) + 0.5)
            blin = lin[b.bl] + mu * a[k]
            hb, wb = blin.shape
            idx = np.arange(hb * wb).reshape(hb, wb)
            pi, pj, cap = [], [], []
            for t, (dy, dx) in enumerate(spec.dirs[:nf]):
                ys, xs = slice(0, hb - max(0, dy)), slice(max(0, -dx), wb - max(0, dx))
                yt, xt = slice(dy, hb - max(0, dy) + dy), slice(max(0, -dx) + dx, wb - max(0, dx) + dx)
                wq = (b.wd[t] / (q * spec.shift(q, dy, dx, 1.0)))[b.bl]
                wsel = wq[ys, xs]
                m = wsel != 0
                pi.append(idx[ys, xs][m])
                pj.append(idx[yt, xt][m])
                cap.append(lam * wsel[m])
            pi = np.concatenate(pi).astype(np.int32)
            pj = np.concatenate(pj).astype(np.int32)
            cap = np.concatenate(cap)
            labels, _ = orc.bk_maxflow(blin.ravel(), pi, pj, cap, cap)
            yh[k] = np.asarray(labels, dtype=np.int8).reshape(hb, wb)
        # ---- global step (admm.py:136-180) ----
        acc = np.zeros((H, W))
        for k, b in enumerate(blocks):
            q = b.q
            t = np.zeros(q.shape)
            t[b.bl] = yh[k]
            accw = acc[b.win]
            accw[b.bl] += mu * (yh[k] + a[k]) - lam * (b.rdiag[b.bl] * yh[k])
            ct = np.where(b.inbox, (b.deg / q) * (1.0 - 1.0 / q) * t, 0.0)
            for ((dy, dx), w), (nb_in, nq) in zip(zip(spec.dirs, b.wd), b.nin):
                # contribution of neighbour i = p + off to pixel p: c_k[i, p] yhat_i
                ti = spec.shift(t, dy, dx)
                ct += np.where(nb_in, np.where(b.inbox, (-w / nq) * (1.0 - 1.0 / q), -w / nq) * ti, 0.0)
            accw -= lam * ct
        y = acc / (mu * spec.q)
        clamped = bool((y < 0).any() or (y > 1).any())
        y = np.clip(y, 0.0, 1.0)
        # ---- residuals, energy, trace, best, multipliers, stop ----
        res = np.array([math.sqrt(float(np.sum((yh[k] - y[b.win][b.bl]) ** 2))) for k, b in enumerate(blocks)])
        e = float(np.sum(spec.u * y))
        for t, (dy, dx) in enumerate(spec.dirs[:nf]):
            e += lam * float(np.sum(spec.wd[t] * (y - spec.shift(y, dy, dx)) ** 2))
        tr["mu"].append(mu)
        tr["energy"].append(e)
        tr["residual_sq"].append(float(np.dot(res, res)))
        tr["max_block_residual"].append(float(res.max()))
        tr["clamped"].append(clamped)
        if e < best_e:
            best_e, best_y, best_it = e, y.copy(), it
        for k, b in enumerate(blocks):
            a[k] = a[k] + (yh[k] - y[b.win][b.bl])
        mu *= mu_fact
        if res.max() <= eps:
            converged = True
            break
    yfin = y if converged else best_y
    return dict(y=yfin.ravel(), labels=(yfin.ravel() >= 0.5).astype(np.int8), iterations=it,
                converged=converged, best_iteration=best_it,
                a_copies=np.concatenate([x.ravel() for x in a]),
                yhat_copies=np.concatenate([x.ravel() for x in yh]),
                **{k: np.array(v) for k, v in tr.items()})
