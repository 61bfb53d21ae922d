"""Sharded (multi-GPU) protocol on one GPU with virtual ranks: the slab /
ghost-row / all-reduce path must reproduce the single-GPU run bit-for-bit
(energies, max residuals, labels); residual_sq is summed per shard (rtol)."""
import numpy as np
import pytest

import paper_1704_03116_b200 as dope
from paper_1704_03116_b200 import sharded, workloads as W
from conftest import load_golden

pytestmark = pytest.mark.gpu


def _model(wl):
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u.astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    return model, part


@pytest.mark.parametrize("shards", [2, 3, 4])
def test_virtual_shards_match_reference_c1(shards):
    g = load_golden("run_c1.npz")
    wl = W.c1()
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=int(g["max_iters"]))
    labels, trace, st = sharded.run_virtual(model, part, cfg, shards)
    assert st["iterations"] == int(g["iterations"])
    assert st["best_iteration"] == int(g["best_iteration"])
    assert np.array_equal([t.energy for t in trace], g["energy"])
    assert np.array_equal([t.max_block_residual for t in trace], g["max_block_residual"])
    np.testing.assert_allclose([t.residual_sq for t in trace], g["residual_sq"], rtol=1e-12)
    assert np.array_equal([t.clamped for t in trace], g["clamped"])
    assert np.array_equal(st["y"], g["y"])
    assert np.array_equal(labels, g["labels"])


@pytest.mark.parametrize("size,block,shards", [(1024, 64, 4), (1024, 64, 16), (512, 128, 4)])
def test_virtual_shards_match_single_gpu(size, block, shards):
    wl = W.disks_workload("s", size, 16, block, 2, 12, rmin=10, rmax=150, seed=3)
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    labels1, s1 = dope.run(model, part, cfg)
    labels, trace, st = sharded.run_virtual(model, part, cfg, shards)
    assert st["iterations"] == s1.iteration
    assert [t.energy for t in trace] == [t.energy for t in s1.trace]
    assert [t.max_block_residual for t in trace] == [t.max_block_residual for t in s1.trace]
    assert np.array_equal(labels, labels1)
    assert np.array_equal(st["yhat"], s1.labels_global())


def test_nccl_single_rank_graph_matches_single_gpu():
    """The C++/NCCL sharded loop (captured in one CUDA graph) with world = 1."""
    import os
    import torch.distributed as dist
    wl = W.mini_disks(256, 64, 8, 2, 25, seed=1)
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    labels1, s1 = dope.run(model, part, cfg)
    comm = sharded.NcclComm(0, 1)
    try:
        sh = sharded.shard_for_rank(model, part, cfg, 0, 1)
        sh.run(comm, cfg.max_iters, use_graph=True)
        labels, trace, st = sharded.collect([sh], 1.0, cfg)
    finally:
        comm.close()
    assert [t.energy for t in trace] == [t.energy for t in s1.trace]
    assert np.array_equal(labels, labels1)
    assert st["best_iteration"] == s1.best_iteration


@pytest.mark.parametrize("size,block,shards", [(96, 32, 3), (128, 32, 2), (64, 16, 4)])
def test_virtual_3d_shards_match_single_gpu(size, block, shards):
    """3D: slabs of block planes with ghost planes (C4's multi-GPU layout)."""
    wl = W.c4(seed=4, size=size, block=block, iters=10)
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    labels1, s1 = dope.run(model, part, cfg)
    labels, trace, st = sharded.run_virtual(model, part, cfg, shards)
    assert st["iterations"] == s1.iteration
    assert [t.energy for t in trace] == [t.energy for t in s1.trace]
    assert [t.max_block_residual for t in trace] == [t.max_block_residual for t in s1.trace]
    np.testing.assert_allclose([t.residual_sq for t in trace], [t.residual_sq for t in s1.trace], rtol=1e-12)
    assert [t.clamped for t in trace] == [t.clamped for t in s1.trace]
    assert np.array_equal(labels, labels1)
    assert np.array_equal(st["yhat"], s1.labels_global())
    assert np.array_equal(st["y"], s1.y)


def test_nccl_single_rank_graph_matches_single_gpu_3d():
    wl = W.c4(seed=6, size=64, block=32, iters=12)
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    labels1, s1 = dope.run(model, part, cfg)
    comm = sharded.NcclComm(0, 1)
    try:
        sh = sharded.shard_for_rank(model, part, cfg, 0, 1)
        sh.run(comm, cfg.max_iters, use_graph=True)
        labels, trace, st = sharded.collect([sh], 1.0, cfg)
    finally:
        comm.close()
    assert [t.energy for t in trace] == [t.energy for t in s1.trace]
    assert np.array_equal(labels, labels1)
    assert st["best_iteration"] == s1.best_iteration
