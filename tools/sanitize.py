"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize.py [case ...]

Cases (each a few ADMM iterations through the public API):
  k1k2_2d     C1-like 256^2, 64^2 blocks: K1 64x64 + the consensus kernels
  tma_list    2304^2, 64^2 blocks (1296 > 2 x CTAs): K1 solved list + TMA K2 phases A/B
  small2d     128^2, 16^2 blocks: K1 16x16 + the warp consensus pass
  k1_3d       64^3, 32^3 blocks: shared-memory K1-3D + plane-mapped K2-3D
  float2d     C2-like 128^2 float weights: K1f / K2f
  general2d   overlap 25 %, mu_fact 1.05: K1g / global step
  graph3d     3D overlap: the general graph path (gstep + batched max-flow)
  loopback    2 loopback shards: ghost consensus, halo copies, decide
  bk          seam 1: one general graph
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_03116_b200 as dope  # noqa: E402
from paper_1704_03116_b200 import sharded, workloads as W  # noqa: E402


def model_of(wl, overlap=0):
    rows, cols, vals = wl.pair_arrays()
    u = wl.u.astype(np.float64)
    model = dope.EnergyModel(u, dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, overlap)
    return model, part


def cfg(it, mu=1.0, fact=1.0):
    return dope.AdmmConfig(mu0=mu, mu_fact=fact, eps=0.0, max_iters=it)


def case_k1k2_2d():
    m, p = model_of(W.mini_disks(256, 64, 6, 2, 4, seed=1))
    return dope.run(m, p, cfg(4))


def case_tma_list():
    m, p = model_of(W.disks_workload("t", 2304, 16, 64, 2, 3, rmin=10, rmax=150, seed=2))
    return dope.run(m, p, cfg(3))


def case_small2d():
    m, p = model_of(W.mini_disks(128, 16, 4, 2, 4, seed=3, rmax=30.0))
    return dope.run(m, p, cfg(4))


def case_k1_3d():
    m, p = model_of(W.c4(seed=4, size=64, block=32, iters=3))
    return dope.run(m, p, cfg(3))


def case_float2d():
    wl = W.c2(size=128, block=64, iters=3)
    m, p = model_of(wl)
    return dope.run(m, p, cfg(3, mu=wl.rho))


def case_general2d():
    wl = W.c2(size=64, block=16, iters=3)
    m, p = model_of(wl, overlap=25)
    return dope.run(m, p, dope.AdmmConfig(max_iters=3, eps=0.0))


def case_graph3d():
    wl = W.c4(seed=5, size=16, block=8, iters=2)
    m, p = model_of(wl, overlap=25)
    return dope.run(m, p, cfg(2))


def case_loopback():
    wl = W.mini_disks(256, 32, 6, 2, 3, seed=6)
    m, p = model_of(wl)
    return sharded.run_virtual(m, p, cfg(3), 2)


def case_bk():
    rng = np.random.default_rng(1)
    m = 40
    pairs = [(i, j) for i in range(m) for j in range(i + 1, m) if rng.random() < 0.2]
    pi = np.array([a for a, _ in pairs], dtype=np.int32)
    pj = np.array([b for _, b in pairs], dtype=np.int32)
    return dope.bk_maxflow(rng.uniform(-3, 3, m), pi, pj, rng.random(pi.size), rng.random(pi.size))


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}


def main(argv):
    torch.cuda.set_device(0)
    names = argv or list(CASES)
    for nm in names:
        CASES[nm]()
        torch.cuda.synchronize()
        print(f"ok {nm}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
