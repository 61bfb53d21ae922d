"""Diagnostics: per pass, how many blocks the 2D TMA consensus pass (K2)
handles in full / ring-only / settled mode (recomputed from the stamps it
keeps, dirty[K, 7K)), and the eager K2 time.  Run on the GPU box:
    python tools/k2_modes.py [C3] [iters]"""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from bench import build_problem
from paper_1704_03116_b200 import workloads as W
from paper_1704_03116_b200.admm import _DeviceState

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
wl = W.by_name(cfg)
_, _, problems = build_problem(wl, torch.device("cuda", 0))
dev = _DeviceState(problems, int(wl.rho), 0.0, iters, True, True)
K = wl.num_blocks
KY, KX = wl.kpa
dev.call("dope_admm_init")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(iters):
    dev.call("dope_update_blocks")
    torch.cuda.synchronize()
    d = dev.dirty.cpu().numpy().astype(np.int64)
    rs = dev.run_state()
    cur, best = rs.ycur, rs.ybest
    out = 3 - cur - best if cur != best else (cur + 1) % 3
    ep = d[K:2 * K] == it + 1
    epg = ep.reshape(KY, KX)
    sd = np.zeros((KY, KX), bool)
    sd[:, 1:] |= epg[:, :-1]
    sd[:, :-1] |= epg[:, 1:]
    sd[1:, :] |= epg[:-1, :]
    sd[:-1, :] |= epg[1:, :]
    ych = d[5 * K:6 * K].reshape(KY, KX)
    ok = (d[6 * K:7 * K].reshape(KY, KX) == it) & (ych < it)
    okr = np.ones((KY, KX), bool)
    okr[:, :-1] = ych[:, 1:] < it
    okd = np.ones((KY, KX), bool)
    okd[:-1, :] = ych[1:, :] < it
    so = d[(2 + out) * K:(3 + out) * K].reshape(KY, KX)
    ok = (d[6 * K:7 * K].reshape(KY, KX) == it) & (so != 0) & (so >= ych) & ~epg & (it >= 2)
    ev[0].record()
    dev.call("dope_update_global", fuse=1)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"pass {it:3d} cur {cur} best {best} out {out}: solved {int(ep.sum()):5d} ring {int((ok & sd).sum()):5d} "
          f"settled {int((ok & ~sd).sum()):5d} full-clean {int((~ok & ~epg).sum()):5d}  K2 {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us")
