"""Anatomy of K1's slowest solves on C3 (diagnostics): for each steady-state
iteration, the slowest blocks' total time split into loads / prologue /
first BFS / the rest, their BFS levels, relabel rounds and sweeps."""
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
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    _, _, problems = build_problem(wl, torch.device("cuda", 0))
    dev = _DeviceState(problems, int(wl.rho), 0.0, iters, True, True)
    K = wl.num_blocks
    # [8K, 16K): per-sweep stamps of a -DK1_DIAG2 build (DOPE_LIB=...)
    t1 = torch.zeros(16 * K + 256, dtype=torch.int64, device="cuda")
    t2 = torch.zeros(8 * K + 64 * K, dtype=torch.int64, device="cuda")
    dev.L.fuse_multipliers = 1
    dev.call("dope_admm_init")
    agg = []
    for it in range(iters):
        t1[: 16 * K].zero_()
        t1[: 8 * K].view(K, 8)[:, 2] = -2
        dev.L.timeline = t1.data_ptr()
        dev.call("dope_update_blocks")
        dev.L.timeline = t2.data_ptr()
        dev.call("dope_update_global", fuse=1)
        torch.cuda.synchronize()
        a = t1[: 8 * K].view(K, 8).cpu().numpy()
        d2 = t1[8 * K: 16 * K].view(K, 8).cpu().numpy()
        solved = np.nonzero(a[:, 2] >= -1)[0]
        if it < 5 or solved.size == 0:
            continue
        dur = (a[solved, 1] - a[solved, 0]) / 1e3
        order = solved[np.argsort(dur)[::-1][:top]]
        med = np.median(dur)
        parts = []
        for k in order:
            r = a[k]
            tot = (r[1] - r[0]) / 1e3
            ld = (r[7] - r[0]) / 1e3
            pro = (r[4] - r[0]) / 1e3
            bfs = (r[5] - r[4]) / 1e3
            rest = (r[1] - r[5]) / 1e3
            rounds, lev_last = r[2] & 0xFFFF, r[2] >> 16
            sweeps, t_last = r[3] & 0xFFFFFF, (r[3] >> 24) / 1e3
            tail = tot - t_last   # last BFS + epilogue
            sw = d2[k]
            if sw[0]:
                cyc = []
                for j in range(3):
                    v = int(sw[j])
                    cyc.append(f"{v & 0xFFFF}/{(v >> 16) & 0xFFFF}/{(v >> 32) & 0xFFFF}/{sw[3 + j]}p{v >> 48}")
                parts.append("[sweep cycles push/bar/relabel/end " + " ".join(cyc) + "]")
            for j, nm in ((6, "bfs1"), (7, "bfs-last")):
                v = int(sw[j])
                if v:
                    parts.append(f"[{nm} masks {v & 0xFFFFF} bfs {(v >> 20) & 0xFFFFF} lev {v >> 40}]")
            lev1, nact = r[6] & 0xFFFF, r[6] >> 16
            parts.append(f"{tot:5.1f}us(ld {ld:4.1f} pro {pro:4.1f} bfs1 {bfs:4.1f} lev {lev1:3d} act {nact:4d} rest {rest:5.1f} "
                         f"rounds {rounds} sweeps {sweeps} last-bfs+epi {tail:4.1f} lev {lev_last})")
            agg.append((tot, ld, pro, bfs, lev1, rest, rounds, sweeps, tail, lev_last, nact))
        print(f"it {it + 1:3d} solved {solved.size:4d} med {med:5.1f} | " + " ".join(parts[:2]))
    A = np.array(agg, dtype=np.float64)
    if A.size:
        print("slowest-block means: total %.1f loads %.1f prologue %.1f bfs1 %.1f levels %.0f rest %.1f rounds %.1f "
              "sweeps %.1f last-bfs+epilogue %.1f last levels %.0f active %.0f" % tuple(A.mean(axis=0)))
        # all solved blocks of the last iteration: rounds / sweeps histogram
    dev.raise_on_error()


if __name__ == "__main__":
    main()
