"""Small driver for ncu captures: one C3 run through the step-level C ABI,
one launch per kernel (no CUDA graph), so each kernel is profiled alone."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import build_problem  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402
from paper_1704_03116_b200.admm import _DeviceState, make_device_state  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    _, _, problems = build_problem(wl, torch.device("cuda", 0))
    if wl.integer:
        dev = _DeviceState(problems, int(wl.rho), 0.0, iters, True, True)
    else:
        dev = make_device_state(problems, float(wl.rho), 0.0, iters)
    dev.call("dope_admm_init")
    dev.call("dope_admm_run", iters, 0, fuse=1)
    dev.call("dope_finish_run")
    torch.cuda.synchronize()
    rs = dev.raise_on_error()
    print(f"{name}: {rs.iteration} iterations, solves {rs.solves}, sweeps {rs.sweeps}, "
          f"max rounds {rs.max_rounds_seen}, best E {rs.best_energy}")


if __name__ == "__main__":
    main()
