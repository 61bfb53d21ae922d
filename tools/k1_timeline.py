"""Per-block K1 timeline on C3 (diagnostics): which iterations/blocks dominate."""
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
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    _, _, problems = build_problem(wl, torch.device("cuda", 0))
    dev = _DeviceState(problems, int(wl.rho), 0.0, iters, True, True)
    K = wl.num_blocks
    tl = torch.zeros(8 * K, dtype=torch.int64, device="cuda")
    dev.L.timeline = tl.data_ptr()
    dev.call("dope_admm_init")
    for it in range(iters):
        tl.view(K, 8)[:, 2] = -1   # blocks K1 does not solve keep rounds = -1
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        dev.call("dope_update_blocks")
        e1.record()
        t = tl.view(K, 8).cpu().numpy()   # before the consensus pass writes its own diagnostics
        dev.call("dope_update_global", fuse=1)
        e2.record()
        torch.cuda.synchronize()
        solved = t[:, 2] >= 0
        t0 = t[solved, 0].min() if solved.any() else 0
        dur = (t[:, 1] - t[:, 0]) / 1e3
        ends = (t[solved, 1] - t0) / 1e3 if solved.any() else np.zeros(1)
        starts = (t[solved, 0] - t0) / 1e3 if solved.any() else np.zeros(1)
        ds = dur[solved]
        print(f"it {it+1:3d}: K1 {e0.elapsed_time(e1)*1e3:7.1f} us  K2 {e1.elapsed_time(e2)*1e3:6.1f} us | "
              f"solved {solved.sum():5d}  block us: med {np.median(ds) if ds.size else 0:6.1f} "
              f"p90 {np.percentile(ds,90) if ds.size else 0:6.1f} max {ds.max() if ds.size else 0:6.1f} | "
              f"last start {starts.max():6.1f} last end {ends.max():6.1f} | rounds max {t[:,2].max()} "
              f"sweeps med {np.median(t[solved,3]) if solved.any() else 0:.0f} max {t[:,3].max()}")
        if solved.any():
            pro = (t[solved, 4] - t[solved, 0]) / 1e3
            ld = (t[solved, 7] - t[solved, 0]) / 1e3
            bfs = (t[solved, 5] - t[solved, 4]) / 1e3
            rest = (t[solved, 1] - t[solved, 5]) / 1e3
            lev = t[solved, 6] & 0xFFFF
            print(f"        loads med {np.median(ld):5.1f} max {ld.max():5.1f} | prologue med {np.median(pro):5.1f} max {pro.max():5.1f} | bfs1 med {np.median(bfs):5.1f} "
                  f"max {bfs.max():5.1f} levels med {np.median(lev):.0f} max {lev.max()} | rest med {np.median(rest):5.1f} "
                  f"max {rest.max():5.1f}")
    rs = dev.raise_on_error()
    print("state", rs.iteration, rs.best_energy)


if __name__ == "__main__":
    main()
