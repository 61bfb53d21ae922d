"""Diagnostics: does a C4 block's last solve time predict its next one?
(K1-3D runs in two waves when more than 148 blocks are dirty; longest-first
dispatch would need a predictor.)"""
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
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    torch.cuda.set_device(0)
    wl = W.by_name("C4")
    _, _, problems = build_problem(wl, torch.device("cuda", 0))
    dev = _DeviceState(problems, int(wl.rho), 0.0, iters, True, True)
    K = wl.num_blocks
    tl = torch.zeros(8 * K, dtype=torch.int64, device="cuda")
    dev.L.timeline = tl.data_ptr()
    dev.call("dope_admm_init")
    last = np.full(K, np.nan)
    pairs = []
    for it in range(iters):
        tl.view(K, 8)[:, 2] = -1
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.call("dope_update_blocks")
        e1.record()
        dev.call("dope_update_global", fuse=1)
        torch.cuda.synchronize()
        t = tl.view(K, 8).cpu().numpy()
        s = np.flatnonzero(t[:, 2] >= 0)
        dur = (t[s, 1] - t[s, 0]) / 1e3
        if it >= 3:
            prev = last[s]
            ok = ~np.isnan(prev)
            pairs += list(zip(prev[ok], dur[ok]))
            order = np.argsort(-dur)
            # ideal LPT makespan on 148 SMs vs arrival order (list scheduling)
            def makespan(d):
                slots = np.zeros(148)
                for x in d:
                    i = int(np.argmin(slots))
                    slots[i] += x
                return slots.max()
            pred = np.where(np.isnan(prev), np.nanmedian(last), prev)
            print(f"it {it+1:3d}: solved {s.size:4d} K1 {e0.elapsed_time(e1)*1e3:6.1f} us | block med {np.median(dur):5.1f} "
                  f"max {dur.max():5.1f} | makespan arrival {makespan(dur):6.1f} LPT-true {makespan(dur[order]):6.1f} "
                  f"LPT-predicted {makespan(dur[np.argsort(-pred)]):6.1f} | rounds max {t[s,2].max()}")
        last[s] = dur
    p = np.array(pairs)
    print("corr(last solve, next solve) =", np.corrcoef(p[:, 0], p[:, 1])[0, 1], "n =", len(p))


if __name__ == "__main__":
    main()
