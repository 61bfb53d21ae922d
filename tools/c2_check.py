"""C2 float parity detail: GPU vs oracle at full 1024^2 size (first N iterations)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402

import oracle as orc  # noqa: E402
import paper_1704_03116_b200 as dope  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
wl = W.c2(iters=iters)
rows, cols, vals = wl.pair_arrays()
model = dope.EnergyModel(wl.u, dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)
part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
labels, st = dope.run(model, part, dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=iters))
spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, wl.weights, wl.u, wl.lam)
ref = orc.run(spec, wl.rho, 1.0, 0.0, iters, threads=16)
e = np.array([t.energy for t in st.trace])
print("iterations", st.iteration, ref["iterations"], "best", st.best_iteration, ref["best_iteration"])
print("max rel energy diff per iteration", np.max(np.abs(e - ref["energy"]) / np.abs(ref["energy"])))
print("final energy rel diff", abs(e[-1] - ref["energy"][-1]) / abs(ref["energy"][-1]))
print("label disagreement", int((labels != ref["labels"]).sum()), "of", labels.size)
print("block-label disagreement (last it)", int((st.labels_global() != ref["yhat"]).sum()))
