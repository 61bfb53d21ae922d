"""Per-CTA timeline of the persistent TMA consensus pass (diagnostics):
CTA start / end spread and the last-CTA finalize tail."""
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
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    torch.cuda.set_device(0)
    wl = W.by_name(name)
    _, _, problems = build_problem(wl, torch.device("cuda", 0))
    dev = _DeviceState(problems, int(wl.rho), 0.0, iters, True, True)
    K = wl.num_blocks
    tl = torch.zeros(8 * K, dtype=torch.int64, device="cuda")
    dev.L.timeline = tl.data_ptr()
    dev.call("dope_admm_init")
    G = torch.cuda.get_device_properties(0).multi_processor_count
    for it in range(iters):
        dev.call("dope_update_blocks")
        tl.zero_()
        e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e1.record()
        dev.call("dope_update_global", fuse=1)
        e2.record()
        torch.cuda.synchronize()
        t = tl.view(K, 8).cpu().numpy()
        ncta = min(4 * G, K)   # the TMA pass's persistent grid
        st = t[:ncta, 6][t[:ncta, 6] > 0]
        en = t[:, 7][: len(st)]
        if st.size == 0:
            print(f"it {it+1}: no TMA timeline (generic consensus path)")
            continue
        t0 = st.min()
        fin = t[len(st), 7] if len(st) < K else 0
        print(f"it {it+1:3d}: K2 {e1.elapsed_time(e2)*1e3:6.1f} us | ctas {len(st)} start spread "
              f"{(st.max()-t0)/1e3:5.1f} us | end min {(en.min()-t0)/1e3:5.1f} med {(np.median(en)-t0)/1e3:5.1f} "
              f"max {(en.max()-t0)/1e3:5.1f} us | finalize end {(fin-t0)/1e3 if fin else float('nan'):5.1f} us")
        if it == iters - 1 and (t[: len(st), 0] > 0).any():
            # per-CTA detail (TMA pass slots: 0 metadata, 1 last issue, 4 stages, 5 phase-A blocks)
            c = t[: len(st)]
            meta = (c[:, 0] - c[:, 6]) / 1e3
            print(f"  metadata gathered after: med {np.median(meta):.1f} max {meta.max():.1f} us")
            for nst in sorted(set(c[:, 4].tolist())):
                m = c[:, 4] == nst
                print(f"  {int(m.sum()):4d} CTAs with {nst:2d} stages: end med {(np.median(c[m, 7]) - t0)/1e3:5.1f} "
                      f"max {(c[m, 7].max() - t0)/1e3:5.1f} us, phase-A blocks {np.bincount(c[m, 5]).tolist()}")
            G = len(st)
            if K < 5 * G:   # no room for the per-stage stamps
                continue
            sg = tl.cpu().numpy()[8 * G: 8 * G + 32 * G].reshape(G, 8, 4)
            for b in np.argsort(c[:, 7])[-3:].tolist() + [int(np.argsort(c[:, 7])[G // 2])]:
                ns = int(c[b, 4])
                rows = [f"({(sg[b, i, 0] - t0)/1e3:.1f},{(sg[b, i, 1] - t0)/1e3:.1f},{(sg[b, i, 3] - t0)/1e3:.1f},{(sg[b, i, 2] - t0)/1e3:.1f})"
                        for i in range(min(ns, 8))]
                print(f"  CTA {b}: start {(c[b, 6] - t0)/1e3:.1f} meta {(c[b, 0] - t0)/1e3:.1f} stages "
                      f"[issue,data,loop,done] {' '.join(rows)} drained {(c[b, 2] - t0)/1e3:.1f} end {(c[b, 7] - t0)/1e3:.1f}")
    dev.raise_on_error()


if __name__ == "__main__":
    main()
