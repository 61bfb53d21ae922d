"""GPU parity: the B200 path vs the reference's golden traces and the oracle.

Integer configs must be bit-exact every iteration: block labels, energies,
max block residual, clamped flag, final y / labels / multipliers.
residual_sq is a float sum of sqrt(int)^2 (admm.py:237) whose summation order
is BLAS-specific in the reference, so it is compared at rtol 1e-12.
"""
import os

import numpy as np
import pytest

import paper_1704_03116_b200 as dope
from paper_1704_03116_b200 import _lib, workloads as W
from conftest import golden_cases, load_golden, spec_from_golden

pytestmark = pytest.mark.gpu

CASES_ALL = [c for c in golden_cases() if not c.startswith("c2")]   # integer configs


def model_from_golden(g):
    dims = tuple(int(d) for d in g["dims"])
    if "kpa" in g:
        kpa = tuple(int(k) for k in g["kpa"])
    else:
        kpa = tuple(d // int(b) for d, b in zip(dims, g["block"]))
    wl = W.Workload("g", dims, (1, 1), int(g["conn"]), g["u"], [1.0] * (2 if len(dims) == 2 else 3),
                    float(g["lam"]), float(g["rho"]), int(g["max_iters"]), True)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(g["u"].astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             float(g["lam"]))
    part = dope.make_partition(dope.GridShape(dims), kpa, 0)
    return model, part


def test_library_is_the_cuda_build():
    lb = _lib.lib()
    assert lb.dope_backend_name() == b"b200-sm100a"
    import torch
    assert torch.cuda.is_available()


@pytest.mark.parametrize("opts", [dict(warm_start=True, skip_clean=True, use_graph=True),
                                  dict(warm_start=False, skip_clean=False, use_graph=False),
                                  dict(warm_start=True, skip_clean=False, use_graph=True),
                                  dict(warm_start=False, skip_clean=True, use_graph=False)])
@pytest.mark.parametrize("case", CASES_ALL)
def test_run_matches_reference_trace(case, opts):
    g = load_golden(f"run_{case}.npz")
    model, part = model_from_golden(g)
    cfg = dope.AdmmConfig(mu0=float(g["rho"]), mu_fact=1.0, eps=0.0,
                          max_iters=int(g["max_iters"]), **opts)
    labels, state = dope.run(model, part, cfg)
    assert state.iteration == int(g["iterations"])
    assert state.converged == bool(g["converged"])
    assert state.best_iteration == int(g["best_iteration"])
    e = np.array([t.energy for t in state.trace])
    assert np.array_equal(e, g["energy"])
    assert np.array_equal([t.max_block_residual for t in state.trace], g["max_block_residual"])
    np.testing.assert_allclose([t.residual_sq for t in state.trace], g["residual_sq"], rtol=1e-12)
    assert np.array_equal([t.clamped for t in state.trace], g["clamped"])
    assert np.array_equal([t.mu for t in state.trace], g["mu"])
    assert np.array_equal(state.y, g["y"])
    assert np.array_equal(labels, g["labels"])
    assert np.array_equal(state.multipliers_global(), g["a"])
    hist = np.unpackbits(g["yhat_bits"], axis=1)[:, :model.n]
    assert np.array_equal(state.labels_global(), hist[-1])


@pytest.mark.parametrize("case", ["c1", "mini128_b16", "ragged", "mini3d"])
def test_step_api_block_labels_every_iteration(case):
    """The public step functions (general graph path on the device) reproduce the
    reference's run iteration by iteration."""
    g = load_golden(f"run_{case}.npz")
    model, part = model_from_golden(g)
    problems = dope.assemble_block_problems(model, part)
    cfg = dope.AdmmConfig(mu0=float(g["rho"]), mu_fact=1.0, eps=0.0, max_iters=int(g["max_iters"]))
    state = dope.init_state(part, float(g["rho"]))
    hist = np.unpackbits(g["yhat_bits"], axis=1)[:, :model.n]
    for it in range(int(g["iterations"])):
        dope.update_blocks(state, problems, model.lam, cfg)
        assert np.array_equal(state.labels_global(), hist[it]), it
        dope.update_global(state, problems, part, model.lam)
        assert state.clamped_last == bool(g["clamped"][it])
        res = dope.block_residuals(state, part)
        assert float(res.max()) == g["max_block_residual"][it]
        assert dope.evaluate_energy(model, state.y) == g["energy"][it]
        dope.update_multipliers(state, part, 1.0)


@pytest.mark.parametrize("case", ["c1", "mini128_b16", "ragged", "mini3d"])
def test_abi_step_entries_every_iteration(case):
    """The lattice ABI's step entries (dope_update_blocks / dope_update_global /
    dope_update_multipliers, include/dope_b200.h) driven one call at a time."""
    from paper_1704_03116_b200.admm import make_device_state
    g = load_golden(f"run_{case}.npz")
    model, part = model_from_golden(g)
    problems = dope.assemble_block_problems(model, part)
    assert problems.kind == "int"
    dev = make_device_state(problems, float(g["rho"]), 0.0, int(g["max_iters"]))
    dev.call("dope_admm_init")
    hist = np.unpackbits(g["yhat_bits"], axis=1)[:, :model.n]
    for it in range(int(g["iterations"])):
        dev.call("dope_update_blocks")
        dev.raise_on_error()
        assert np.array_equal(dev.yhat.cpu().numpy(), hist[it]), it
        dev.call("dope_update_global", fuse=0)
        dev.dirty[2 * len(problems):].zero_()   # step calls keep no clean-block stamps
        assert bool(dev.pf.any().item()) == bool(g["clamped"][it])
        ss = dev.pr.cpu().numpy()
        assert float(np.sqrt(ss.max())) == g["max_block_residual"][it]
        dev.call("dope_update_multipliers")
    assert np.array_equal(dev.a.double().cpu().numpy(), g["a"])


def test_bk_maxflow_seam_matches_reference_graphs():
    g = load_golden("bk_graphs.npz")
    mo, po = g["m_off"], g["p_off"]
    mism = 0
    for k in range(len(mo) - 1):
        sm, sp = slice(mo[k], mo[k + 1]), slice(po[k], po[k + 1])
        tcap, cij, cji = g["tcap"][sm], g["cij"][sp], g["cji"][sp]
        lab, flow = dope.bk_maxflow(tcap, g["pi"][sp], g["pj"][sp], cij, cji)
        integral = np.all(tcap == np.round(tcap)) and np.all(cij == np.round(cij)) \
            and np.all(cji == np.round(cji))
        assert flow == pytest.approx(g["flows"][k], abs=1e-9), k
        if integral:
            assert np.array_equal(lab, g["labels"][sm]), k
        else:
            mism += int(not np.array_equal(lab, g["labels"][sm]))
    assert mism == 0


def test_bk_maxflow_reference_known_answers():
    lab, flow = dope.bk_maxflow(np.array([-1.0]), [], [], [], [])
    assert lab.tolist() == [1] and flow == 0.0
    lab, flow = dope.bk_maxflow(np.array([2.0, -1.0, 0.0, -0.5]), [], [], [], [])
    assert lab.tolist() == [0, 1, 0, 1]
    g = dope.FlowGraph(2)
    g.add_terminal(0, 4.0, 0.0)
    g.add_terminal(1, 0.0, 4.0)
    g.add_edge(0, 1, 1.0, 10.0)
    labels, flow = dope.min_cut(g)
    assert flow == pytest.approx(1.0) and labels.tolist() == [0, 1]
    w = dope.SparseWeights(4, [0, 1, 2], [1, 2, 3], [1.0, 1.0, 1.0])
    labels, flow = dope.solve_binary(np.zeros(4), w, 1.0)
    assert flow == 0.0 and len(set(labels.tolist())) == 1


@pytest.mark.parametrize("size,block,iters", [(1024, 64, 8), (512, 32, 8), (512, 128, 6),
                                               (2560, 64, 10)])
def test_larger_grids_match_oracle(size, block, iters):
    """(2560, 64): 1600 blocks, more than two per consensus CTA, so the TMA pass
    deals out K1's solved-block list and takes its settled / ring-only paths."""
    import oracle as orc
    wl = W.disks_workload(f"t{size}", size, 16, block, 2, iters, rmin=10, rmax=150, seed=11)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u.astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=iters)
    labels, state = dope.run(model, part, cfg)
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, [1.0, 1.0], wl.u.astype(np.float64),
                           wl.lam)
    ref = orc.run(spec, 1.0, 1.0, 0.0, iters, threads=8)
    assert state.iteration == ref["iterations"]
    assert np.array_equal([t.energy for t in state.trace], ref["energy"])
    assert np.array_equal([t.max_block_residual for t in state.trace], ref["max_block_residual"])
    assert np.array_equal(state.y, ref["y"])
    assert np.array_equal(labels, ref["labels"])
    assert np.array_equal(state.labels_global(), ref["yhat"])


def _c3_model():
    wl = W.c3()
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u.astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    return wl, model, part


def test_c3_full_size_first_iterations_match_oracle():
    """BASELINE's 4096^2 grid at full size: first 6 iterations bit-exact vs the oracle
    (from the third on, the consensus pass settles clean blocks from its stamps)."""
    import oracle as orc
    wl, model, part = _c3_model()
    iters = 6
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=iters)
    labels, state = dope.run(model, part, cfg)
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, [1.0, 1.0], wl.u.astype(np.float64), wl.lam)
    ref = orc.run(spec, 1.0, 1.0, 0.0, iters, threads=16)
    assert np.array_equal([t.energy for t in state.trace], ref["energy"])
    assert np.array_equal([t.max_block_residual for t in state.trace], ref["max_block_residual"])
    assert np.array_equal(state.labels_global(), ref["yhat"])
    assert np.array_equal(labels, ref["labels"])


def test_c3_full_run_properties():
    """Full 100-iteration C3 run: deterministic, best-iterate energy consistent with the
    returned labels (size-independent properties)."""
    wl, model, part = _c3_model()
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    labels1, s1 = dope.run(model, part, cfg)
    labels2, s2 = dope.run(model, part, dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0,
                                                         max_iters=wl.iters, use_graph=False,
                                                         skip_clean=False, warm_start=False))
    assert np.array_equal(labels1, labels2)
    assert [t.energy for t in s1.trace] == [t.energy for t in s2.trace]
    assert [t.max_block_residual for t in s1.trace] == [t.max_block_residual for t in s2.trace]
    assert np.allclose([t.residual_sq for t in s1.trace], [t.residual_sq for t in s2.trace], rtol=1e-12, atol=0)
    assert [t.clamped for t in s1.trace] == [t.clamped for t in s2.trace]
    assert np.array_equal(s1.y, s2.y)
    assert np.array_equal(s1.labels_global(), s2.labels_global())
    assert np.array_equal(s1.multipliers_global(), s2.multipliers_global())
    e = [t.energy for t in s1.trace]
    assert s1.best_iteration == int(np.argmin(e)) + 1
    # the returned state.y is the best iterate (binary on the int path): its energy is the min
    assert dope.evaluate_energy(model, s1.y) == min(e)


@pytest.mark.parametrize("size,block,iters", [(96, 32, 6), (64, 16, 8)])
def test_3d_grids_match_oracle(size, block, iters):
    import oracle as orc
    wl = W.c4(seed=21, size=size, block=block, iters=iters)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u.astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    labels, state = dope.run(model, part, dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0,
                                                          max_iters=iters))
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, [1.0, 1.0, 1.0], wl.u.astype(np.float64),
                           wl.lam)
    ref = orc.run(spec, 1.0, 1.0, 0.0, iters, threads=16)
    assert state.iteration == ref["iterations"]
    assert np.array_equal([t.energy for t in state.trace], ref["energy"])
    assert np.array_equal(state.labels_global(), ref["yhat"])
    assert np.array_equal(labels, ref["labels"])


@pytest.mark.parametrize("size,kpa,lam,uscale,iters", [
    (96, (3, 3, 3), 3.0, 1, 6),        # 32^3 boxes, 2cap = 12: shared-memory K1-3D
    (80, (3, 3, 3), 1.0, 1, 8),        # ragged 27/27/26 boxes inside the 32^3 layout
    (64, (2, 2, 2), 1.0, 5000, 5),     # |2u| > 32000 - 6cap: per-block HBM-scratch fallback
    (64, (2, 2, 2), 4.0, 1, 5),        # 2cap = 16 > 15: HBM-scratch kernel
    (64, (4, 2, 2), 2.0, 1, 6),        # mixed 16/32 box extents
])
def test_3d_k1_paths_match_oracle(size, kpa, lam, uscale, iters):
    import oracle as orc
    wl = W.c4(seed=5, size=size, block=size // kpa[0], iters=iters)
    u = wl.u.astype(np.float64)
    if uscale != 1:   # a few slabs of huge unaries: only their blocks leave int16 excess
        u3 = u.reshape(wl.dims).copy()
        u3[: size // 2] *= uscale
        u = u3.ravel()
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(u, dope.SparseWeights(wl.n, rows, cols, vals), lam)
    part = dope.make_partition(dope.GridShape(wl.dims), kpa, 0, materialize=False)
    labels, state = dope.run(model, part, dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=iters))
    spec = orc.LatticeSpec(wl.dims, kpa, wl.offsets, [1.0, 1.0, 1.0], u, lam)
    ref = orc.run(spec, 1.0, 1.0, 0.0, iters, threads=16)
    assert state.iteration == ref["iterations"]
    assert np.array_equal([t.energy for t in state.trace], ref["energy"])
    assert np.array_equal(state.labels_global(), ref["yhat"])
    assert np.array_equal(labels, ref["labels"])


def test_c4_full_size_first_iterations_match_oracle():
    """C4 at full size, 5 iterations bit-exact vs the oracle (from the third on the
    consensus pass settles clean blocks and recomputes only re-solved-neighbour faces)."""
    import oracle as orc
    iters = 5
    wl = W.c4(iters=iters)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u.astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    labels, state = dope.run(model, part, dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=iters))
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, [1.0, 1.0, 1.0], wl.u.astype(np.float64), wl.lam)
    ref = orc.run(spec, 1.0, 1.0, 0.0, iters, threads=os.cpu_count() or 16)
    assert np.array_equal([t.energy for t in state.trace], ref["energy"])
    assert np.array_equal([t.max_block_residual for t in state.trace], ref["max_block_residual"])
    assert np.array_equal(state.labels_global(), ref["yhat"])
    assert np.array_equal(labels, ref["labels"])


def test_c4_clean_block_paths_match_plain_run():
    """C4, 30 iterations: the clean-block consensus paths (settled / face-only
    recompute, memoised energies and clamp groups) against a run that re-solves and
    recomputes every block every iteration -- identical traces, iterates, labels."""
    iters = 30
    wl = W.c4(iters=iters)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u.astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    l1, s1 = dope.run(model, part, dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=iters))
    l2, s2 = dope.run(model, part, dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=iters,
                                                   skip_clean=False))
    assert [t.energy for t in s1.trace] == [t.energy for t in s2.trace]
    assert [t.max_block_residual for t in s1.trace] == [t.max_block_residual for t in s2.trace]
    assert [t.clamped for t in s1.trace] == [t.clamped for t in s2.trace]
    assert np.allclose([t.residual_sq for t in s1.trace], [t.residual_sq for t in s2.trace], rtol=1e-12, atol=0)
    assert np.array_equal(s1.y, s2.y) and np.array_equal(l1, l2)
    assert np.array_equal(s1.labels_global(), s2.labels_global())
    assert np.array_equal(s1.multipliers_global(), s2.multipliers_global())


def _float_model(wl):
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u, dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    return model, part


def test_float_c2mini_matches_reference_within_tolerance():
    """C2-like float config vs the reference trace: BASELINE's bar is final energy
    within 1e-5 relative and <= 0.01 % label disagreement; we also check every
    iteration's energy and the block labels."""
    g = load_golden("run_c2mini.npz")
    wl = W.c2(size=128, block=32, iters=int(g["max_iters"]))
    assert np.array_equal(wl.u, g["u"])
    model, part = _float_model(wl)
    cfg = dope.AdmmConfig(mu0=float(g["rho"]), mu_fact=1.0, eps=0.0, max_iters=int(g["max_iters"]))
    labels, state = dope.run(model, part, cfg)
    e = np.array([t.energy for t in state.trace])
    np.testing.assert_allclose(e, g["energy"], rtol=1e-5)
    assert abs(e[-1] - g["energy"][-1]) <= 1e-5 * abs(g["energy"][-1])
    assert np.mean(labels != g["labels"]) <= 1e-4
    hist = np.unpackbits(g["yhat_bits"], axis=1)[:, :model.n]
    assert np.mean(state.labels_global() != hist[state.iteration - 1]) <= 1e-4


@pytest.mark.parametrize("size,block,iters", [(256, 64, 20), (512, 64, 10)])
def test_float_grids_match_oracle_within_tolerance(size, block, iters):
    import oracle as orc
    wl = W.c2(seed=5, size=size, block=block, iters=iters)
    model, part = _float_model(wl)
    labels, state = dope.run(model, part, dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0,
                                                          max_iters=iters))
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, wl.weights, wl.u, wl.lam)
    ref = orc.run(spec, wl.rho, 1.0, 0.0, iters, threads=16)
    e = np.array([t.energy for t in state.trace])
    np.testing.assert_allclose(e, ref["energy"], rtol=1e-5)
    assert np.mean(labels != ref["labels"]) <= 1e-4


@pytest.mark.parametrize("size,block", [(512, 64), (250, 62)])
def test_float_energy_prepass_equals_the_consensus_pass_sum(size, block, monkeypatch):
    """dope_lattice_f.energy_prepass (K1f sums a re-solved block's interior energy
    while warp 0 runs the relabel BFS) against the consensus pass's own loop:
    identical labels and iterates, energies equal up to summation order."""
    from paper_1704_03116_b200 import admm as A
    wl = W.c2(seed=7, size=size, block=block, iters=16)
    model, part = _float_model(wl)
    cfg = dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=16)
    runs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("DOPE_F_EPRE", flag)
        A._forget(A._problems_for(model, part))   # new device state for each setting
        labels, state = dope.run(model, part, cfg)
        assert A._problems_for(model, part)._run_dev.L.energy_prepass == int(flag)
        runs.append((labels, state.labels_global().copy(), np.array(state.y).copy(),
                     np.array([t.energy for t in state.trace])))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])
    assert np.array_equal(runs[0][2], runs[1][2])
    np.testing.assert_allclose(runs[0][3], runs[1][3], rtol=1e-12)


def test_float_run_variants_agree_with_energy_prepass():
    """Float path with the K1f energy prepass: eager vs graph launches, cold vs
    warm solves and clean-block skipping on / off give the same labels, iterates
    and (up to summation order) energies."""
    wl = W.c2(seed=9, size=256, block=64, iters=14)
    model, part = _float_model(wl)
    base = None
    for kw in ({}, {"use_graph": False}, {"warm_start": False}, {"skip_clean": False}):
        cfg = dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=14, **kw)
        labels, state = dope.run(model, part, cfg)
        got = (labels, state.labels_global().copy(), np.array(state.y).copy(),
               np.array([t.energy for t in state.trace]))
        if base is None:
            base = got
            continue
        assert np.array_equal(got[0], base[0]), kw
        assert np.array_equal(got[1], base[1]), kw
        assert np.array_equal(got[2], base[2]), kw
        np.testing.assert_allclose(got[3], base[3], rtol=1e-12, err_msg=str(kw))
