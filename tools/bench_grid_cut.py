"""Whole-grid serial cut (compare mode) timings: GPU dope_gc_mincut vs the
oracle's BK (host, one thread) on the same models."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_03116_b200 as dope  # noqa: E402
from paper_1704_03116_b200 import compare, workloads as W  # noqa: E402


def model_of(wl):
    rows, cols, vals = wl.pair_arrays()
    return dope.EnergyModel(np.asarray(wl.u, dtype=np.float64), dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)


def main():
    import oracle as orc
    out = {}
    for name, wl in (("C2 1024^2 8-conn float", W.c2()), ("C5 2048^2 4-conn int", W.c5(64)),
                     ("C3 4096^2 4-conn int", W.c3())):
        m = model_of(wl)
        compare.solve_binary_grid(m.unary, m.weights, m.lam, wl.dims)   # warm-up (allocator, module load)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lab, flow = compare.solve_binary_grid(m.unary, m.weights, m.lam, wl.dims)
        torch.cuda.synchronize()
        gpu = time.perf_counter() - t0
        rec = {"gpu_s": gpu, "pixels": wl.n, "pairs": m.weights.npairs}
        if wl.n <= 4_200_000:
            w = m.weights
            t1 = time.perf_counter()
            ref, _ = orc.bk_maxflow(m.unary.copy(), w.rows.astype(np.int32), w.cols.astype(np.int32),
                                    m.lam * w.vals, m.lam * w.vals)
            rec["bk_host_s"] = time.perf_counter() - t1
            rec["label_diff"] = int(np.count_nonzero(np.asarray(ref, dtype=np.int8) != lab))
        out[name] = rec
    print(json.dumps(out))


if __name__ == "__main__":
    main()
