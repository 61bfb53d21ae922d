"""Diagnostics: does a pinned H2D on a side stream overlap a DOPE run?"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from bench import build_problem  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402
from paper_1704_03116_b200.admm import make_device_state  # noqa: E402

wl = W.by_name("C3")
_, _, problems = build_problem(wl, torch.device("cuda", 0))
dev = make_device_state(problems, wl.rho, 0.0, 100, True, True)
comp, cs = torch.cuda.Stream(), torch.cuda.Stream()
host = problems.u.cpu().pin_memory()
dst = torch.empty_like(problems.u)
ev = lambda: torch.cuda.Event(enable_timing=True)


def run():
    with torch.cuda.stream(comp):
        dev.call("dope_admm_init")
        dev.call("dope_admm_run", 100, 1, fuse=1)
        dev.call("dope_finish_run")


run(); torch.cuda.synchronize()
for trial in range(3):
    t0, a0, a1, b0, b1 = ev(), ev(), ev(), ev(), ev()
    t0.record(comp)
    cs.wait_event(t0)
    a0.record(comp)
    run()
    a1.record(comp)
    b0.record(cs)
    with torch.cuda.stream(cs):
        dst.copy_(host, non_blocking=True)
    b1.record(cs)
    torch.cuda.synchronize()
    print(f"compute {t0.elapsed_time(a0):.2f}->{t0.elapsed_time(a1):.2f} ms | copy {t0.elapsed_time(b0):.2f}->{t0.elapsed_time(b1):.2f} ms")
