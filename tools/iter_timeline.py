"""Whole-iteration timeline on C3 (diagnostics): K1 per-block start / end and
the consensus pass's per-CTA start / end on one globaltimer axis, launched
back to back on one stream like the run loop.  Shows where an iteration's
time goes: K1 ramp, slowest solve, the K1 -> K2 gap, K2's CTA spread.

    python tools/iter_timeline.py [config] [iterations] [print-from]
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
    t1 = torch.zeros(8 * K, dtype=torch.int64, device="cuda")
    t2 = torch.zeros(8 * K + 64 * K, dtype=torch.int64, device="cuda")
    dev.L.fuse_multipliers = 1   # the run loop's mode (dirty-block worklists)
    dev.call("dope_admm_init")
    G = torch.cuda.get_device_properties(0).multi_processor_count
    rows = []
    for it in range(iters):
        t1.view(K, 8)[:, 2] = -2
        t2.zero_()
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        dev.L.timeline = t1.data_ptr()
        dev.call("dope_update_blocks")
        e1.record()
        dev.L.timeline = t2.data_ptr()
        dev.call("dope_update_global", fuse=1)
        e2.record()
        torch.cuda.synchronize()
        a = t1.view(K, 8).cpu().numpy()
        b = t2[: 8 * K].view(K, 8).cpu().numpy()
        solved = a[:, 2] >= -1
        ncta = min(4 * G, K)
        cs = b[:ncta, 6]
        ok = cs > 0
        if not solved.any() or not ok.any():
            continue
        t0 = a[solved, 0].min()
        k1_end = a[solved, 1]
        k2s, k2e = cs[ok], b[:ncta, 7][ok]
        r = dict(it=it + 1, k1_ev=e0.elapsed_time(e1) * 1e3, k2_ev=e1.elapsed_time(e2) * 1e3,
                 solved=int(solved.sum()),
                 k1_last_start=(a[solved, 0].max() - t0) / 1e3,
                 k1_med_end=(np.median(k1_end) - t0) / 1e3, k1_p90_end=(np.percentile(k1_end, 90) - t0) / 1e3,
                 k1_last_end=(k1_end.max() - t0) / 1e3,
                 k2_first=(k2s.min() - t0) / 1e3, k2_med_end=(np.median(k2e) - t0) / 1e3,
                 k2_last_end=(k2e.max() - t0) / 1e3,
                 med_solve=float(np.median((a[solved, 1] - a[solved, 0]) / 1e3)),
                 max_solve=float(((a[solved, 1] - a[solved, 0]) / 1e3).max()))
        rows.append(r)
        if it + 1 >= show:
            print(f"it {r['it']:3d} ev K1 {r['k1_ev']:5.1f} K2 {r['k2_ev']:5.1f} | solved {r['solved']:4d} "
                  f"solve med {r['med_solve']:5.1f} max {r['max_solve']:5.1f} | K1 last start {r['k1_last_start']:5.1f} "
                  f"end med {r['k1_med_end']:5.1f} p90 {r['k1_p90_end']:5.1f} last {r['k1_last_end']:5.1f} | "
                  f"K2 first {r['k2_first']:5.1f} end med {r['k2_med_end']:5.1f} last {r['k2_last_end']:5.1f}")
    st = [r for r in rows if r["it"] > 5]
    if st:
        keys = ["k1_ev", "k2_ev", "solved", "med_solve", "max_solve", "k1_last_start", "k1_med_end", "k1_p90_end",
                "k1_last_end", "k2_first", "k2_med_end", "k2_last_end"]
        print("mean over iterations > 5:", {k: round(float(np.mean([r[k] for r in st])), 2) for k in keys})
    dev.raise_on_error()


if __name__ == "__main__":
    main()
