"""The sharded (multi-GPU) run loop of csrc/dope_comm.cu on one GPU.

The loopback communicator holds all G shards of one grid in this process and
drives the SAME C++ iteration and graph capture as NCCL (one label-halo
exchange, dope_ghost_consensus, one gather of the exact integer agg slots,
dope_decide); each boundary row moves by one cudaMemcpyAsync.  Every trace
field (residual_sq included: the agg slots are exact integers), the labels,
the iterate and the per-iteration state digests must equal the single-GPU
run and the oracle's full-length fixtures bit for bit, for G = 2, 4, 8 on the
benchmarked configs.  The NCCL communicator itself runs at world size 1.
"""
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


def _same_run(trace, st, labels, s1, labels1):
    assert st["iterations"] == s1.iteration
    assert st["best_iteration"] == s1.best_iteration
    assert st["converged"] == s1.converged
    assert [t.energy for t in trace] == [t.energy for t in s1.trace]
    assert [t.max_block_residual for t in trace] == [t.max_block_residual for t in s1.trace]
    assert [t.residual_sq for t in trace] == [t.residual_sq for t in s1.trace]
    assert [t.clamped for t in trace] == [t.clamped for t in s1.trace]
    assert np.array_equal(labels, labels1)
    assert np.array_equal(st["yhat"], s1.labels_global())
    assert np.array_equal(st["y"], s1.y)
    assert np.array_equal(st["a"], s1.multipliers_global())


@pytest.mark.parametrize("shards", [2, 3, 4])
def test_loopback_shards_match_reference_c1(shards):
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
    assert np.array_equal(st["a"], g["a"])


@pytest.mark.parametrize("size,block,shards,graph,peer", [(1024, 64, 4, True, False), (1024, 64, 16, True, False),
                                                           (512, 128, 4, True, False), (1024, 64, 8, False, False),
                                                           (1024, 64, 4, True, True), (1024, 64, 16, True, True),
                                                           (512, 128, 4, False, True)])
def test_loopback_shards_match_single_gpu(size, block, shards, graph, peer):
    wl = W.disks_workload("s", size, 16, block, 2, 30, rmin=10, rmax=150, seed=3)
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    labels1, s1 = dope.run(model, part, cfg)
    labels, trace, st = sharded.run_virtual(model, part, cfg, shards, use_graph=graph, peer=peer)
    _same_run(trace, st, labels, s1, labels1)


@pytest.mark.parametrize("name,shards,peer", [("C3", 2, False), ("C3", 4, False), ("C3", 8, False),
                                              ("C5-B64", 8, False), ("C4", 2, False), ("C4", 4, False),
                                              ("C4", 8, False), ("C3", 8, True), ("C4", 8, True)])
def test_loopback_full_size_matches_fixture_every_iteration(name, shards, peer):
    """BASELINE configs at full size and full length, sharded G ways (copies
    between kernels, or the peer-memory exchange): the summed per-shard digests
    equal the oracle's every iteration."""
    g = load_golden(f"full_{name.lower()}.npz")
    wl = W.by_name(name)
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    labels, trace, st = sharded.run_virtual(model, part, cfg, shards, digests=True, peer=peer)
    it = int(g["iterations"])
    assert st["iterations"] == it
    assert st["best_iteration"] == int(g["best_iteration"])
    assert np.array_equal([t.energy for t in trace], g["energy"])
    assert np.array_equal([t.max_block_residual for t in trace], g["max_block_residual"])
    assert np.array_equal([t.clamped for t in trace], g["clamped"])
    np.testing.assert_allclose([t.residual_sq for t in trace], g["residual_sq"], rtol=1e-12)
    bad = [t + 1 for t in range(it) if not np.array_equal(st["digests"][t], g["digests"][t])]
    assert not bad, f"digests differ at iterations {bad[:10]}"


@pytest.mark.parametrize("size,block,shards,peer", [(96, 32, 3, False), (128, 32, 2, False), (64, 16, 4, False),
                                                    (96, 32, 3, True), (64, 16, 4, True)])
def test_loopback_3d_shards_match_single_gpu(size, block, shards, peer):
    """3D: slabs of block planes with ghost planes (C4's multi-GPU layout)."""
    wl = W.c4(seed=4, size=size, block=block, iters=20)
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    labels1, s1 = dope.run(model, part, cfg)
    labels, trace, st = sharded.run_virtual(model, part, cfg, shards, peer=peer)
    _same_run(trace, st, labels, s1, labels1)


def test_loopback_graph_cache_released_with_the_communicator():
    from paper_1704_03116_b200 import _lib
    wl = W.mini_disks(256, 32, 8, 2, 10, seed=2)
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    lb = _lib.lib()
    lb.dope_graph_cache_clear()
    for _ in range(3):
        sharded.run_virtual(model, part, cfg, 4)
    assert lb.dope_graph_cache_entries() == 0   # each group's graph died with its communicator


@pytest.mark.parametrize("three_d", [False, True])
def test_nccl_single_rank_graph_matches_single_gpu(three_d):
    """The C++/NCCL sharded loop (captured in one CUDA graph) with world = 1."""
    wl = W.c4(seed=6, size=64, block=32, iters=12) if three_d else W.mini_disks(256, 64, 8, 2, 25, seed=1)
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
    _same_run(trace, st, labels, s1, labels1)


def test_ipc_peer_comm_single_rank_matches_single_gpu():
    """The multi-GPU peer-memory transport (CUDA IPC handles, library-owned
    buffers) at world size 1: export / init path and the peer-mode loop."""
    wl = W.mini_disks(256, 64, 8, 2, 20, seed=5)
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    labels1, s1 = dope.run(model, part, cfg)
    sh = sharded.shard_for_rank(model, part, cfg, 0, 1, ipc=True)
    comm = sharded.IpcPeerComm(sh)
    try:
        sh.run(comm, cfg.max_iters, use_graph=True)
        labels, trace, st = sharded.collect([sh], 1.0, cfg)
    finally:
        comm.close()
    _same_run(trace, st, labels, s1, labels1)
