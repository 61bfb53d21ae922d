"""World-size-2 gloo test of the multi-GPU protocol on CPU.

Two processes each own a slab of block rows; run_shards + DistComm drive the
label halo and the agg all-gather over gloo; the shards compute with the CPU
test executor (tests/cpu_shard.py), which recomputes the ghost rows' iterate
locally like dope_ghost_consensus.  The assembled result must equal the
single-domain oracle run (itself pinned to the reference) bit-for-bit --
residual_sq included (the exact integer agg slots).  The product C++ loop
(csrc/dope_comm.cu) runs the same protocol; tests/test_sharded_gpu.py drives
it through the loopback communicator on one GPU.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from cpu_shard import CpuShardND
    from paper_1704_03116_b200 import sharded
    u, dims, kpa, lamw, iters = case
    slabs = sharded.shard_block_rows(kpa[0], world)
    kb0, kb1 = slabs[rank]
    sh = CpuShardND(u, dims, kpa, lamw, 1, iters, kb0, kb1, index=rank, count=world)
    sharded.run_shards([sh], sharded.DistComm(), iters)
    np.savez(Path(out_dir) / f"rank{rank}.npz", labels=sh.labels(), energy=np.array(sh.trace_e),
             maxres=np.array(sh.trace_mr), rs=np.array(sh.trace_rs), it=sh.it,
             best=sh.best_it, conv=sh.converged)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_rank_sharded_run_matches_oracle(world, tmp_path):
    import oracle as orc
    from paper_1704_03116_b200 import workloads as W
    wl = W.mini_disks(64, 16, 4, 2, 6, seed=9, rmax=24.0)
    case = (wl.u, wl.dims, wl.kpa, int(wl.lam), wl.iters)
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, [1.0, 1.0], wl.u.astype(np.float64), wl.lam)
    ref = orc.run(spec, 1.0, 1.0, 0.0, wl.iters)
    labels = np.concatenate([o["labels"].ravel() for o in outs])
    for o in outs:   # every rank made the same decisions
        assert int(o["it"]) == ref["iterations"]
        assert int(o["best"]) == ref["best_iteration"]
        assert np.array_equal(o["energy"], ref["energy"])
        assert np.array_equal(o["maxres"], ref["max_block_residual"])
        np.testing.assert_allclose(o["rs"], ref["residual_sq"], rtol=1e-12)
    assert np.array_equal(labels, ref["labels"])


@pytest.mark.parametrize("world", [3])
def test_gloo_three_rank_sharded_run_matches_oracle(world, tmp_path):
    """A middle rank with ghost rows on both sides; 40 iterations (blocks 8 rows deep)."""
    import oracle as orc
    from paper_1704_03116_b200 import workloads as W
    wl = W.mini_disks(48, 8, 5, 2, 40, seed=4, rmax=14.0)
    case = (wl.u, wl.dims, wl.kpa, int(wl.lam), wl.iters)
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, [1.0, 1.0], wl.u.astype(np.float64), wl.lam)
    ref = orc.run(spec, 1.0, 1.0, 0.0, wl.iters)
    labels = np.concatenate([o["labels"].ravel() for o in outs])
    for o in outs:
        assert int(o["it"]) == ref["iterations"]
        assert int(o["best"]) == ref["best_iteration"]
        assert np.array_equal(o["energy"], ref["energy"])
        assert np.array_equal(o["maxres"], ref["max_block_residual"])
        np.testing.assert_allclose(o["rs"], ref["residual_sq"], rtol=1e-14)
    assert np.array_equal(labels, ref["labels"])


@pytest.mark.parametrize("world", [2])
def test_gloo_two_rank_sharded_run_3d_matches_oracle(world, tmp_path):
    """3D (C4's layout): slabs of block planes, ghost-plane halos over gloo."""
    import oracle as orc
    from paper_1704_03116_b200 import workloads as W
    wl = W.c4(seed=8, size=16, block=8, iters=6)
    case = (wl.u, wl.dims, wl.kpa, int(wl.lam), wl.iters)
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, [1.0, 1.0, 1.0], wl.u.astype(np.float64), wl.lam)
    ref = orc.run(spec, 1.0, 1.0, 0.0, wl.iters)
    labels = np.concatenate([o["labels"].ravel() for o in outs])
    for o in outs:
        assert int(o["it"]) == ref["iterations"]
        assert int(o["best"]) == ref["best_iteration"]
        assert np.array_equal(o["energy"], ref["energy"])
        assert np.array_equal(o["maxres"], ref["max_block_residual"])
        np.testing.assert_allclose(o["rs"], ref["residual_sq"], rtol=1e-12)
    assert np.array_equal(labels, ref["labels"])
