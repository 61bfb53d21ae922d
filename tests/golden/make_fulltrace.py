"""Full-length trace fixtures of the BASELINE configs, made by the CPU oracle.

TEST INFRASTRUCTURE ONLY.  For every BASELINE.json config at full size and full
iteration count (C1 50, C2 100, C3 100, C4 60, C5 b16/b32/b64/b128 100) this runs
the oracle's restatement of admm.run (oracle/dope_oracle.c, itself pinned
bit-for-bit to traces the reference produced, tests/test_oracle_golden.py) on the
seeded workload of paper_1704_03116_b200.workloads and stores, per iteration:

  energy, residual_sq, max_block_residual, clamped, mu        (admm.py:233-241)
  digest[t] = state_digest(yhat_t, y_t, a_t)                  (3 x uint64)

plus the final iterations / converged / best_iteration, the digest of the
returned state (final yhat, state.y = best iterate, final multipliers), a digest
of the returned binary labels and a checksum of the input unary (so a test can
prove it regenerated the same workload).  The digests are the order-independent
position-weighted sums of dope_oracle.c:state_digest, which the device computes
per iteration when dope_lattice.trace_hash is set (tests/test_full_traces.py).

For the float config C2 only the yhat digest is meaningful (y and a are not
integers); the file also keeps the final labels as packed bits for the
BASELINE tolerance bar (<= 0.01 % labels, final energy within 1e-5).

Usage:  python tests/golden/make_fulltrace.py [C1 C3 ...]   (default: all)
Runtime on 8 host cores: about 20 minutes for all eight configs.
"""
from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as orc  # noqa: E402  (checker)
from paper_1704_03116_b200 import workloads as W  # noqa: E402

CONFIGS = ["C1", "C2", "C3", "C4", "C5-B16", "C5-B32", "C5-B64", "C5-B128"]


def u_checksum(u: np.ndarray) -> np.uint64:
    """Position-weighted checksum of the unary (int64 view of u*2, or its float bits)."""
    z = np.zeros(u.size, dtype=np.uint8)
    if np.all(u == np.round(u)):
        return orc.state_digest(z, u.astype(np.float64) / 2.0, np.zeros(u.size))[1]
    bits = np.ascontiguousarray(u, dtype=np.float64).view(np.int64)
    return np.uint64(int(bits.astype(np.uint64).sum(dtype=np.uint64)))


def make(name: str, threads: int) -> Path:
    wl = W.by_name(name)
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, wl.weights if not wl.integer
                           else [1.0] * len(wl.offsets), wl.u.astype(np.float64), wl.lam)
    t0 = time.time()
    out = orc.run(spec, wl.rho, 1.0, 0.0, wl.iters, threads=threads, digests=True)
    dt = time.time() - t0
    rec = dict(
        name=np.array(wl.name), dims=np.array(wl.dims), kpa=np.array(wl.kpa),
        iters=np.int32(wl.iters), integer=np.bool_(wl.integer),
        u_checksum=np.uint64(u_checksum(wl.u)),
        energy=out["energy"], residual_sq=out["residual_sq"],
        max_block_residual=out["max_block_residual"], clamped=out["clamped"], mu=out["mu"],
        digests=out["digests"], iterations=np.int32(out["iterations"]),
        converged=np.bool_(out["converged"]), best_iteration=np.int32(out["best_iteration"]),
        final_digest=orc.state_digest(out["yhat"], out["y"], out["a"]),
        labels_digest=orc.state_digest(out["labels"].astype(np.uint8), np.zeros(wl.n),
                                       np.zeros(wl.n))[0],
        oracle_seconds=np.float64(dt), oracle_threads=np.int32(threads),
    )
    if not wl.integer:
        rec["labels_bits"] = np.packbits(out["labels"].astype(np.uint8))
        rec["yhat_bits"] = np.packbits(out["yhat"])
    path = HERE / f"full_{wl.name.lower()}.npz"
    np.savez_compressed(path, **rec)
    print(f"{wl.name}: {out['iterations']} iterations in {dt:.0f} s -> {path.name}", flush=True)
    return path


def main(argv):
    names = [a.upper() for a in argv] or CONFIGS
    threads = os.cpu_count() or 8
    for nm in names:
        make(nm, threads)


if __name__ == "__main__":
    main(sys.argv[1:])
