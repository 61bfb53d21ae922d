"""Throughput of the GPU model builders on a 4096^2 RGB
image, kernel 3 (8-connected): pairs/s and achieved HBM GB/s of the weight
kernel (algorithmic bytes: 2 x 3 x 8 B of colour reads + 24 B of rows/cols/
vals writes per pair), unary pixels/s; the reference's numpy builders timed on
a 512^2 crop on the host for comparison."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1704_03116_b200 as dope  # noqa: E402
from paper_1704_03116_b200 import _lib, inputs as din  # noqa: E402
import ctypes as C  # noqa: E402


def main():
    n_side = 4096
    rng = np.random.default_rng(0)
    data = rng.uniform(0, 1, (n_side * n_side, 3))
    shape = dope.GridShape((n_side, n_side))
    img = din.GridImage(shape, data)
    dev = torch.device("cuda", 0)
    offs, dims, noff = din._window(shape, 3)
    lb = _lib.lib()
    po = offs.ctypes.data_as(C.POINTER(C.c_int32))
    total = int(lb.dope_in_pair_count(2, dims, noff, po))
    d = torch.as_tensor(data, device=dev)
    rows = torch.empty(total, dtype=torch.int64, device=dev)
    cols = torch.empty_like(rows)
    vals = torch.empty(total, dtype=torch.float64, device=dev)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        lb.dope_in_potts_weights(2, dims, 3, d.data_ptr(), noff, po, 0.1, 1, rows.data_ptr(), cols.data_ptr(),
                                 vals.data_ptr(), s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        lb.dope_in_potts_weights(2, dims, 3, d.data_ptr(), noff, po, 0.1, 1, rows.data_ptr(), cols.data_ptr(),
                                 vals.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    alg = total * (2 * 3 * 8 + 24)
    cm = din.ColorModel(rng.uniform(0, 1, (5, 3)), rng.uniform(0, 1, (5, 3)), np.full(5, 0.2), np.full(5, 0.2), 0.2)
    t0 = time.perf_counter()
    din.compute_unaries(img, cm)
    torch.cuda.synchronize()
    t_u = time.perf_counter() - t0
    # reference-style numpy on a 512^2 crop (host)
    sys.path.insert(0, "/root/reference/pkg/src")
    host = None
    try:
        from dope.energy import build_potts_weights as ref_bpw
        from dope.grid import GridImage as RefImage, GridShape as RefShape
        crop = RefImage(RefShape((512, 512)), data[: 512 * 512])
        t1 = time.perf_counter()
        ref_bpw(crop, 3, 0.1)
        host = (512 * 512 * 4) / (time.perf_counter() - t1)
    except Exception as exc:   # the reference is not on GPU boxes
        host = f"unavailable ({type(exc).__name__})"
    print(json.dumps({"pairs": total, "weights_ms": ms, "pairs_per_s": total / (ms / 1e3),
                      "weights_GBps": alg / (ms / 1e3) / 1e9, "unaries_incl_h2d_s": t_u,
                      "host_numpy_pairs_per_s_512crop": host}))


if __name__ == "__main__":
    main()
