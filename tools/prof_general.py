"""Eager general-path run (one launch per kernel, no graph) for ncu captures."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import general_model  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402
from paper_1704_03116_b200.general import GeneralDevice, lower_general  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2-ov25"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    model, part = general_model(wl)
    low = lower_general(model, part)
    gd = GeneralDevice(low, wl.meta["mu0"], wl.meta["mu_fact"], 0.0, iters)
    gd.init()
    for _ in range(iters):
        gd.step_blocks()
        gd.step_global()
    torch.cuda.synchronize()
    print(name, "iterations", gd.run_state().iteration)


if __name__ == "__main__":
    main()
