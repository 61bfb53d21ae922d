import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_1704_03116_b200 as dope
from paper_1704_03116_b200 import workloads as W
import oracle as orc
for frac in (0, 32, 64):
    size, kpa, lam, iters = 64, (2,2,2), 1.0, 5
    wl = W.c4(seed=5, size=size, block=32, iters=iters)
    u3 = wl.u.astype(np.float64).reshape(wl.dims).copy()
    u3[:frac] *= 5000
    u = u3.ravel()
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(u, dope.SparseWeights(wl.n, rows, cols, vals), lam)
    part = dope.make_partition(dope.GridShape(wl.dims), kpa, 0, materialize=False)
    labels, state = dope.run(model, part, dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=iters))
    spec = orc.LatticeSpec(wl.dims, kpa, wl.offsets, [1.0, 1.0, 1.0], u, lam)
    ref = orc.run(spec, 1.0, 1.0, 0.0, iters, threads=16)
    e = [t.energy for t in state.trace]
    print(frac, os.environ.get("DOPE_K1_3D"), e == list(ref["energy"]), e, list(ref["energy"]),
          int((state.labels_global() != ref["yhat"]).sum()))
