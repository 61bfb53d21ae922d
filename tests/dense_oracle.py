"""Dense restatement of the block operators (TEST INFRASTRUCTURE ONLY).

Straight from the definitions in the reference's blockform.py:1-18 docstring /
the paper's Thm. 1, with dense n x n matrices, for tiny
models: the independent checker of the device step kernels.

  q        block counts, Q = diag(q), W symmetric weights, d = W 1, L = D - W
  S_k      selection of block k's pixels (ascending)
  What_k   = S_k Q^-1 W Q^-1 S_k'        (in-block rescaled weights)
  C_k[i,j] = L[g_i, j] m_j / q_{g_i},  m_j = 1 - 1/q_j inside block k, else 1
  r_k      = d / q^2 (on the block) - What_k 1
  linear_k = S_k u / q + lam (C_k y + r_k * S_k y) + mu (a_k - S_k y + 1/2)
  y*       = (mu Q)^-1 sum_k [S_k' (mu (yhat_k + a_k) - lam r_k * yhat_k) - lam C_k' yhat_k]
  objective(y) = sum_k lam yhat_k . (C_k y + r_k * S_k y) + mu/2 ||S_k y - yhat_k - a_k||^2
"""
import numpy as np


class DenseOps:
    def __init__(self, model, part):
        n = model.n
        w = model.weights
        W = np.zeros((n, n))
        np.add.at(W, (w.rows, w.cols), w.vals)
        np.add.at(W, (w.cols, w.rows), w.vals)
        self.W, self.d = W, W.sum(axis=1)
        self.L = np.diag(self.d) - W
        self.q = np.zeros(n)
        for b in part.blocks:
            self.q[b.pixels] += 1
        self.u, self.lam = model.unary, model.lam
        self.blocks = [b.pixels for b in part.blocks]
        self.C, self.r, self.What = [], [], []
        for p in self.blocks:
            inside = np.zeros(n, dtype=bool)
            inside[p] = True
            m = np.where(inside, 1.0 - 1.0 / self.q, 1.0)
            C = self.L[p, :] / self.q[p][:, None] * m[None, :]
            Wh = W[np.ix_(p, p)] / (self.q[p][:, None] * self.q[p][None, :])
            self.C.append(C)
            self.What.append(Wh)
            self.r.append(self.d[p] / self.q[p] ** 2 - Wh.sum(axis=1))

    def linear(self, k, y, a, mu, lam):
        p = self.blocks[k]
        return self.u[p] / self.q[p] + lam * (self.C[k] @ y + self.r[k] * y[p]) + mu * (a - y[p] + 0.5)

    def solve_global(self, yhat, a, mu, lam):
        acc = np.zeros(self.q.size)
        for k, p in enumerate(self.blocks):
            yh = np.asarray(yhat[k], dtype=np.float64)
            acc[p] += mu * (yh + a[k]) - lam * self.r[k] * yh
            acc -= lam * (self.C[k].T @ yh)
        return acc / (mu * self.q)

    def objective(self, yhat, a, mu, lam, y):
        tot = 0.0
        for k, p in enumerate(self.blocks):
            yh = np.asarray(yhat[k], dtype=np.float64)
            tot += lam * float(yh @ (self.C[k] @ y + self.r[k] * y[p]))
            diff = y[p] - (yh + a[k])
            tot += 0.5 * mu * float(diff @ diff)
        return tot
