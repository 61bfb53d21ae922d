"""Diagnostics: do K1's slowest block solves repeat a recent linear vector?

Runs C3 (or another 2D integer config) iteration by iteration through the
C ABI step entries with the K1 timeline on.  Before each K1 it recomputes
every block's doubled linear term on the host from the device state
(2 lin = 2u + lamw * sum_cross(y2_g - y2_j) + mu (2a - y2 + 1), the q == 1
stencil), and reports per iteration: blocks solved, their solve times, how
many solved blocks' vectors equal one of the last H iterations' vectors, and
what K1's critical path would be if those were memo hits.
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


def lin2_blocks(u, y2, a, dims, block, lamw, mu):
    H, Wd = dims
    bh, bw = block
    y2 = y2.reshape(H, Wd).astype(np.int64)
    s = np.zeros((H, Wd), dtype=np.int64)
    r = np.arange(H)[:, None]
    c = np.arange(Wd)[None, :]
    # cross-block neighbours only
    left = (c % bw == 0) & (c > 0)
    right = (c % bw == bw - 1) & (c < Wd - 1)
    up = (r % bh == 0) & (r > 0)
    down = (r % bh == bh - 1) & (r < H - 1)
    s += np.where(left, y2 - np.roll(y2, 1, axis=1), 0)
    s += np.where(right, y2 - np.roll(y2, -1, axis=1), 0)
    s += np.where(up, y2 - np.roll(y2, 1, axis=0), 0)
    s += np.where(down, y2 - np.roll(y2, -1, axis=0), 0)
    lin = 2 * u.reshape(H, Wd).astype(np.int64) + lamw * s + mu * (2 * a.reshape(H, Wd).astype(np.int64) - y2 + 1)
    return lin.reshape(H // bh, bh, Wd // bw, bw).transpose(0, 2, 1, 3).reshape(-1, bh * bw)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hist_len = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    _, _, problems = build_problem(wl, torch.device("cuda", 0))
    dev = _DeviceState(problems, int(wl.rho), 0.0, iters, True, True)
    K = wl.num_blocks
    tl = torch.zeros(8 * K, dtype=torch.int64, device="cuda")
    dev.L.timeline = tl.data_ptr()
    dev.call("dope_admm_init")
    u = wl.u
    lamw, mu = problems.lowering.lamw, int(wl.rho)
    history = []
    tot_solved = tot_rep = 0
    k1_sum = k1_memo_sum = 0.0
    for it in range(iters):
        y2 = dev.y2_current().cpu().numpy()
        a = dev.a.cpu().numpy()
        lin = lin2_blocks(u, y2, a, wl.dims, wl.block, lamw, mu)
        tl.view(K, 8)[:, 2] = -1
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.call("dope_update_blocks")
        e1.record()
        t = tl.view(K, 8).cpu().numpy()
        dev.call("dope_update_global", fuse=1)
        torch.cuda.synchronize()
        solved = np.flatnonzero(t[:, 2] >= 0)
        dur = (t[:, 1] - t[:, 0]) / 1e3
        rep = np.zeros(K, dtype=bool)
        for h in history:
            rep[solved] |= np.all(h[solved] == lin[solved], axis=1)
        history.append(lin)
        history = history[-hist_len:]
        ds = dur[solved]
        nonrep = solved[~rep[solved]]
        crit = dur[nonrep].max() if nonrep.size else 0.0
        slow = solved[np.argsort(dur[solved])[-max(1, solved.size // 20):]] if solved.size else solved
        k1 = e0.elapsed_time(e1) * 1e3
        if it >= 2:
            tot_solved += solved.size
            tot_rep += int(rep[solved].sum())
            k1_sum += k1
            k1_memo_sum += crit
        print(f"it {it + 1:3d}: K1 {k1:7.1f} us  solved {solved.size:5d} repeats {int(rep[solved].sum()):5d} "
              f"| block us med {np.median(ds) if ds.size else 0:5.1f} max {ds.max() if ds.size else 0:5.1f} "
              f"| slowest 5%: {int(rep[slow].sum())}/{slow.size} repeats | max non-repeat {crit:5.1f} us "
              f"| |lin2| max {int(np.abs(lin[solved]).max()) if solved.size else 0}")
    print(f"iterations 3..{iters}: {tot_rep}/{tot_solved} solved blocks repeat one of the last {hist_len} vectors "
          f"({100.0 * tot_rep / max(tot_solved, 1):.1f} %); K1 sum {k1_sum:.0f} us, max non-repeat block sum "
          f"{k1_memo_sum:.0f} us")


if __name__ == "__main__":
    main()
