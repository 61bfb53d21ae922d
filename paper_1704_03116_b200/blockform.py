"""Per-block subproblems (reference blockform.py:32-105) on the device.

assemble_block_problems returns BlockProblems (admm.py): the lattice lowering
the run-loop kernels use, and -- for the step-level API and any model the
lattice kernels cannot represent -- the general graph path's device data
(graphstep.GraphProblems).  problems[k] is a BlockView with the reference's
BlockProblem fields (block, u_hat, w_hat, d_hat, r_diag, c_rows), computed
on demand; block_objective evaluates the linear term on the device.
"""
from __future__ import annotations

import numpy as np

from .admm import BlockProblems, assemble_block_problems  # noqa: F401  (re-exported)
from .graphstep import BlockView, GraphProblems

BlockProblem = BlockView


def block_objective(bp: BlockView, y, a_k, mu: float, lam: float):
    """(linear, pairwise, scale) of block bp (blockform.py:89-105):
    linear = u_hat + lam (C y + r S y) + mu ((a - S y) + 1/2), on the device."""
    import torch
    if mu < 0 or lam < 0:
        raise ValueError("mu and lambda must be non-negative")
    gp: GraphProblems = bp._p
    lay = gp.layout
    a_k = np.asarray(a_k, dtype=np.float64)
    if a_k.shape != (bp.size,):
        raise ValueError("multiplier length does not match block size")
    e0, e1 = int(lay.blk_ptr[bp.k]), int(lay.blk_ptr[bp.k + 1])
    a = torch.zeros(max(lay.M, 1), dtype=torch.float64, device=gp.device)
    a[e0:e1] = torch.as_tensor(a_k, device=gp.device)
    y = torch.as_tensor(np.ascontiguousarray(y, dtype=np.float64), device=gp.device)
    if tuple(y.shape) != (lay.n,):
        raise ValueError(f"y has shape {tuple(y.shape)}, expected ({lay.n},)")
    lin = gp.objective(y, a, mu, lam, entries=(e0, e1))
    return lin[e0:e1].cpu().numpy(), bp.w_hat, lam
