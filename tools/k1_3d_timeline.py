"""Per-block K1-3D timeline (shared-memory kernel): prologue / relabel / sweeps split."""
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
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
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
        tl.view(K, 8)[:, 2] = -1
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.call("dope_update_blocks")
        e1.record()
        dev.call("dope_update_global", fuse=1)
        torch.cuda.synchronize()
        t = tl.view(K, 8).cpu().numpy()
        s = t[:, 2] >= 0
        if not s.any():
            print(f"it {it+1}: nothing solved")
            continue
        t = t[s]
        t0 = t[:, 0].min()
        dur = (t[:, 1] - t[:, 0]) / 1e3
        pro = (t[:, 4] - t[:, 0]) / 1e3
        bfs = t[:, 7] / 1e3
        swp = dur - pro - bfs
        j = int(np.argmax(dur))
        print(f"it {it+1:3d}: K1 {e0.elapsed_time(e1)*1e3:7.1f} us solved {s.sum():4d} | block us med {np.median(dur):6.1f} "
              f"max {dur.max():7.1f} | last start {(t[:,0].max()-t0)/1e3:6.1f} | prologue med {np.median(pro):5.1f} "
              f"| relabel med {np.median(bfs):6.1f} max {bfs.max():6.1f} lev1 med {np.median(t[:,6]):.0f} max {t[:,6].max()} "
              f"| sweeps-part med {np.median(swp):6.1f} | slowest: rounds {t[j,2]} sweeps {t[j,3]} relabel {bfs[j]:.1f} "
              f"sweeps-part {swp[j]:.1f}")
        if len(sys.argv) > 3 and sys.argv[3] == "diag":   # build with -DK1S_DIAG: [6] passes done [7] bulk copies in
            ps = (t[:, 6] - t[:, 0]) / 1e3
            pl = (t[:, 7] - t[:, 0]) / 1e3
            print(f"        passes done med {np.median(ps):5.1f} max {ps.max():5.1f} | bulk copies in med {np.median(pl):5.1f} "
                  f"max {pl.max():5.1f} | prologue end med {np.median(pro):5.1f}")
    dev.raise_on_error()


if __name__ == "__main__":
    main()
