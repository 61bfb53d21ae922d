"""Anatomy of the float path's block solves on C2 (diagnostics, -DK1F_DIAG
build loaded with DOPE_LIB): per iteration the solved blocks' time split
(prologue / solve / epilogue), relabel rounds, BFS levels, sweeps; from
iteration 12 on also the consensus pass's slowest CTAs (mode, phase stamps).

    nvcc -t 0 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
        -Xcompiler -fPIC -shared -cudart static -Iinclude -Ipaper_1704_03116_b200/csrc \
        -DK1F_DIAG -o paper_1704_03116_b200/libdope_k1fdiag.so paper_1704_03116_b200/csrc/*.cu
    DOPE_LIB=$PWD/paper_1704_03116_b200/libdope_k1fdiag.so python tools/k1f_diag.py C2 24 3
"""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import build_problem  # noqa: E402
from paper_1704_03116_b200 import _lib  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402
from paper_1704_03116_b200.admm import make_device_state  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    _, _, problems = build_problem(wl, torch.device("cuda", 0))
    dev = make_device_state(problems, wl.rho, 0.0, iters, True, True)
    K = wl.num_blocks
    lb = _lib.lib()
    host = np.zeros(16 * K, dtype=np.int64)
    dev.call("dope_admm_init")
    for it in range(iters):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        dev.call("dope_update_blocks")
        e1.record()
        dev.call("dope_update_global", fuse=1)
        e2.record()
        torch.cuda.synchronize()
        lb.dope_f_diag_read(host.ctypes.data_as(C.c_void_p), C.c_int(16 * K))
        h2 = np.zeros(16 * K, dtype=np.int64)
        lb.dope_f_diag_read_k2(h2.ctypes.data_as(C.c_void_p), C.c_int(16 * K))
        b = h2.reshape(K, 16)
        if it >= 12:
            t0k = b[:, 0].min()
            end = np.where(b[:, 7] > 0, b[:, 7], b[:, 1])
            slow = np.argsort(end)[::-1][:3]
            msg = []
            for k in slow:
                x = b[k]
                msg.append(f"[blk {k} mode {x[15]} start {(x[0]-t0k)/1e3:.1f} mode@ {(x[1]-t0k)/1e3:.1f} E {(x[2]-t0k)/1e3:.1f} "
                           f"int {(x[3]-t0k)/1e3:.1f} ring {(x[4]-t0k)/1e3:.1f} red {(x[5]-t0k)/1e3:.1f} "
                           f"tail {(x[6]-t0k)/1e3:.1f} end {(x[7]-t0k)/1e3:.1f}]")
            modes = np.bincount(b[:, 15].astype(int), minlength=5)
            print(f"   K2f modes {modes.tolist()} " + " ".join(msg))
        a = host.reshape(K, 16)
        solved = np.nonzero(a[:, 2] >= a[:, 0] + 1)[0]
        solved = solved[a[solved, 0] > 0]
        # only this iteration's solves: start stamp within this launch
        if solved.size:
            t0 = a[solved, 0].max() - 2_000_000
            solved = solved[a[solved, 0] >= t0]
        if solved.size == 0:
            print(f"it {it}: no solves, K1 {e0.elapsed_time(e1)*1e3:.1f} us K2 {e1.elapsed_time(e2)*1e3:.1f} us")
            continue
        r = a[solved]
        tot = (r[:, 7] - r[:, 0]) / 1e3
        order = np.argsort(tot)[::-1][:top]
        parts = []
        for j in order:
            x = r[j]
            parts.append(f"[{(x[7]-x[0])/1e3:.1f}us pro {(x[1]-x[0])/1e3:.1f} (lin {(x[10]-x[0])/1e3:.1f} bulk {(x[11]-x[10])/1e3:.1f} sync {(x[12]-x[11])/1e3:.1f}) bfs1 {(x[8]-x[1])/1e3:.1f} "
                         f"solve {(x[2]-x[1])/1e3:.1f} epi {(x[7]-x[2])/1e3:.1f} rounds {x[3]} dense {x[6]} "
                         f"lev {x[4]} sw {x[5]} cand {x[9]}]")
        span = (r[:, 7].max() - r[:, 0].min()) / 1e3
        print(f"it {it}: K1 {e0.elapsed_time(e1)*1e3:.1f} us (span {span:.1f}) K2 {e1.elapsed_time(e2)*1e3:.1f} us, "
              f"{solved.size} solves, median {np.median(tot):.1f} us rounds med {np.median(r[:,3]):.0f} "
              f"max {r[:,3].max()} | " + " ".join(parts))


if __name__ == "__main__":
    main()
