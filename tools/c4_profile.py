"""Per-iteration K1/K2 times and solver counters on a 3D config (diagnostics)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import build_problem  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402
from paper_1704_03116_b200.admm import _DeviceState  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    _, _, problems = build_problem(wl, torch.device("cuda", 0))
    for rep in range(2):
        dev = _DeviceState(problems, int(wl.rho), 0.0, iters, True, True)
        dev.call("dope_admm_init")
        torch.cuda.synchronize()
        tk1 = tk2 = 0.0
        prev = (0, 0, 0)
        for it in range(iters):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            dev.call("dope_update_blocks")
            e1.record()
            dev.call("dope_update_global", fuse=1)
            e2.record()
            torch.cuda.synchronize()
            rs = dev.run_state()
            k1, k2 = e0.elapsed_time(e1) * 1e3, e1.elapsed_time(e2) * 1e3
            tk1 += k1
            tk2 += k2
            cur = (rs.solves, rs.sweeps, rs.max_rounds_seen)
            if rep == 1:
                print(f"it {it+1:3d}: K1 {k1:8.1f} us  K2 {k2:6.1f} us  solves {cur[0]-prev[0]:4d} "
                      f"sweeps {cur[1]-prev[1]:8d}  max_rounds {cur[2]}")
            prev = cur
        if rep == 1:
            print(f"total K1 {tk1/1e3:.2f} ms  K2 {tk2/1e3:.2f} ms")
    dev.raise_on_error()


if __name__ == "__main__":
    main()
