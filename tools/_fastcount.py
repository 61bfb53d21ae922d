import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from bench import build_problem
from paper_1704_03116_b200 import workloads as W
from paper_1704_03116_b200.admm import _DeviceState
wl = W.by_name("C4"); _, _, problems = build_problem(wl, torch.device("cuda", 0))
dev = _DeviceState(problems, 1, 0.0, 30, True, True)
K = wl.num_blocks; kp = wl.kpa
dev.call("dope_admm_init")
for it in range(30):
    dev.call("dope_update_blocks")
    torch.cuda.synchronize()
    ep = dev.dirty[K:2*K].cpu().numpy().reshape(kp) == it + 1
    nb = ep.copy()
    for ax in range(3):
        nb |= np.roll(ep, 1, ax) & (np.arange(kp[ax]) > 0).reshape([-1 if a == ax else 1 for a in range(3)])
        nb |= np.roll(ep, -1, ax) & (np.arange(kp[ax]) < kp[ax]-1).reshape([-1 if a == ax else 1 for a in range(3)])
    dev.call("dope_update_global", fuse=1)
    torch.cuda.synchronize()
    if it % 5 == 4: print(it + 1, "solved", ep.sum(), "fast-eligible", (~nb).sum())
