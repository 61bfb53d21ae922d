"""Where the time of one public-API call goes (diagnostics):
run(EnergyModel(u_host_f64, weights, lam), partition, cfg) on a config,
phase by phase with host timers around synchronised sections.

    python tools/public_api_probe.py C3 [steps]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_03116_b200 as dope  # noqa: E402
from paper_1704_03116_b200 import admm as A  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    rows, cols, vals = wl.pair_arrays()
    weights = dope.SparseWeights(wl.n, rows, cols, vals)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0)
    cfg = dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    u_np = np.ascontiguousarray(wl.u, dtype=np.float64)
    for _ in range(3):
        dope.run(dope.EnergyModel(u_np, weights, wl.lam), part, cfg)
    torch.cuda.synchronize()
    tot = []
    for _ in range(steps):
        t0 = time.perf_counter()
        dope.run(dope.EnergyModel(u_np, weights, wl.lam), part, cfg)
        torch.cuda.synchronize()
        tot.append(time.perf_counter() - t0)
    print(f"{name}: public run() {1e3 * np.median(tot):.2f} ms per call ({wl.iters} iterations)")

    # phases
    model = dope.EnergyModel(u_np, weights, wl.lam)
    ph = {}

    def tm(key, fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ph.setdefault(key, []).append(time.perf_counter() - t)
        return r

    for _ in range(steps):
        model = dope.EnergyModel(u_np, weights, wl.lam)
        problems = tm("problems_for (lookup + unary upload)", lambda: A._problems_for(model, part))
        up = problems._uploader
        tm("  upload, registered buffer", lambda: up.upload(u_np))
        tm("  upload, staged (fresh array)", lambda: up.upload(u_np.copy()))
        up.upload(u_np)
        dev = tm("run_state", lambda: problems.run_state(wl.rho, 0.0, cfg))
        tm("device loop (init + run + finish)", lambda: (dev.call("dope_admm_init"),
                                                          dev.call("dope_admm_run", cfg.max_iters, 1, fuse=1),
                                                          dev.call("dope_finish_run")))
        tm("trace reads", lambda: [x[:wl.iters].cpu() for x in (dev.tr_e, dev.tr_rs, dev.tr_mr, dev.tr_cl)])
        tm("labels binarize + D2H", lambda: problems._downloader.fetch(dev.binarize()))
    for k, v in ph.items():
        print(f"  {k:42s} {1e3 * np.median(v):8.3f} ms")
    print(f"uploads: registered {problems._uploader.registered_uploads} staged {problems._uploader.staged_uploads}")
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(steps):
        dope.run(dope.EnergyModel(u_np, weights, wl.lam), part, cfg)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(8)
    pstats.Stats(pr).print_callers("reduce|item|synchronize")


if __name__ == "__main__":
    main()
