"""Time the REFERENCE's own CPU loop (baseline/_ref/dope, staged by
tools/ref_setup.py) on this host -- BASELINE.md §3: the step functions of
admm.run per phase, threads = 1 and threads = nproc, the one-time assembly
separately, CPU model and core count stated.  Writes one JSON line per
(config, threads).

    python tools/time_reference.py C1 C2 [--iters N]
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

import numpy as np  # noqa: E402

import dope  # noqa: E402  (the reference)
from dope import admm as A  # noqa: E402
from dope.blockform import assemble_block_problems  # noqa: E402
from dope.energy import EnergyModel, SparseWeights, evaluate_energy  # noqa: E402
from dope.grid import GridShape  # noqa: E402
from dope.partition import make_partition  # noqa: E402

from bench import cpu_model  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402


def time_config(name, iters, threads):
    wl = W.by_name(name)
    rows, cols, vals = wl.pair_arrays()
    model = EnergyModel(wl.u.astype(np.float64), SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = make_partition(GridShape(wl.dims), wl.kpa, 0)
    t0 = time.perf_counter()
    problems = assemble_block_problems(model, part)
    t_asm = time.perf_counter() - t0
    cfg = A.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=iters, threads=threads)
    state = A.init_state(part, wl.rho)
    ph = {"update_blocks": 0.0, "update_global": 0.0, "block_residuals": 0.0, "evaluate_energy": 0.0,
          "update_multipliers": 0.0}
    t_all = time.perf_counter()
    for _ in range(iters):
        t = time.perf_counter()
        A.update_blocks(state, problems, model.lam, cfg)
        ph["update_blocks"] += time.perf_counter() - t
        t = time.perf_counter()
        A.update_global(state, problems, part, model.lam)
        ph["update_global"] += time.perf_counter() - t
        t = time.perf_counter()
        A.block_residuals(state, part)
        ph["block_residuals"] += time.perf_counter() - t
        t = time.perf_counter()
        evaluate_energy(model, state.y)
        ph["evaluate_energy"] += time.perf_counter() - t
        t = time.perf_counter()
        A.update_multipliers(state, part, 1.0)
        ph["update_multipliers"] += time.perf_counter() - t
    total = time.perf_counter() - t_all
    return {"config": name, "impl": "reference (baseline/_ref/dope, backend " + dope.backend_name() + ")",
            "threads": threads, "nproc": os.cpu_count(), "cpu_model": cpu_model(), "iterations": iters,
            "s_per_iteration": total / iters, "iterations_per_s": iters / total,
            "pixel_edges_per_s": wl.num_pairs * iters / total,
            "phase_s_per_iteration": {k: v / iters for k, v in ph.items()},
            "block_solves_only_it_per_s": iters / ph["update_blocks"],
            "assemble_block_problems_s": t_asm}


def main(argv):
    iters = None
    if "--iters" in argv:
        i = argv.index("--iters")
        iters = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    for name in argv or ["C1", "C2"]:
        n = iters or W.by_name(name).iters
        for threads in (1, os.cpu_count() or 1):
            print(json.dumps(time_config(name, n, threads)), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
