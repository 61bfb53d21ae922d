"""Run-loop iteration timeline (diagnostics): one eager dope_admm_run
iteration at a time, K1's per-block [start, end] and the consensus pass's
per-CTA [start, end] on one globaltimer axis -- in overlap mode both kernels
are live at once (K2's slots follow K1's, consensus_tma.cuh k2_timeline).

    python tools/ovl_timeline.py [config] [iterations] [print-from]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import build_problem  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402
from paper_1704_03116_b200.admm import _DeviceState  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    show = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    _, _, problems = build_problem(wl, torch.device("cuda", 0))
    dev = _DeviceState(problems, int(wl.rho), 0.0, iters, True, True)
    K = wl.num_blocks
    G = torch.cuda.get_device_properties(0).multi_processor_count
    tl = torch.zeros(16 * K + 64 * G, dtype=torch.int64, device="cuda")
    dev.L.timeline = tl.data_ptr()
    dev.call("dope_admm_init")
    rows = []
    for it in range(iters):
        tl.zero_()
        tl[: 8 * K].view(K, 8)[:, 2] = -2
        torch.cuda.synchronize()
        dev.call("dope_admm_run", 1, 0, fuse=1)
        torch.cuda.synchronize()
        a = tl[: 8 * K].view(K, 8).cpu().numpy()
        # K2's per-CTA slots follow K1's in overlap mode, else they overwrite K1's
        ovl = bool((tl[8 * K: 16 * K].view(K, 8)[:, 6] > 0).any())
        b = tl[8 * K: 16 * K].view(K, 8).cpu().numpy() if ovl else None
        solved = a[:, 2] >= -1
        if not solved.any() or b is None:
            print(f"it {it + 1}: solved {solved.sum()} overlap {ovl} (no combined timeline)")
            continue
        t0 = a[solved, 0].min()
        ncta = min(4 * G, K)
        cs, ce = b[:ncta, 6], b[:ncta, 7]
        ok = cs > 0
        k1e = a[solved, 1]
        r = dict(it=it + 1, solved=int(solved.sum()),
                 solve_med=float(np.median((a[solved, 1] - a[solved, 0]) / 1e3)),
                 solve_max=float(((a[solved, 1] - a[solved, 0]) / 1e3).max()),
                 k1_med_end=(np.median(k1e) - t0) / 1e3, k1_last_end=(k1e.max() - t0) / 1e3,
                 k2_first=(cs[ok].min() - t0) / 1e3, k2_med_start=(np.median(cs[ok]) - t0) / 1e3,
                 k2_last_start=(cs[ok].max() - t0) / 1e3,
                 k2_med_end=(np.median(ce[ok]) - t0) / 1e3, k2_last_end=(ce[ok].max() - t0) / 1e3)
        rows.append(r)
        if it + 1 >= show:
            print(f"it {r['it']:3d} solved {r['solved']:4d} solve med {r['solve_med']:5.1f} max {r['solve_max']:5.1f} | "
                  f"K1 end med {r['k1_med_end']:5.1f} last {r['k1_last_end']:5.1f} | K2 start first {r['k2_first']:5.1f} "
                  f"med {r['k2_med_start']:5.1f} last {r['k2_last_start']:5.1f} | end med {r['k2_med_end']:5.1f} "
                  f"last {r['k2_last_end']:5.1f}")
    st = [r for r in rows if r["it"] > 5]
    if st:
        print("mean over iterations > 5:",
              {k: round(float(np.mean([r[k] for r in st])), 2) for k in st[0] if k != "it"})
    dev.raise_on_error()


if __name__ == "__main__":
    main()
