"""Whole-grid serial cut vs the oracle's BK restatement
(itself pinned bit-exact to the reference's compiled core) on full lattices."""
import numpy as np
import pytest

import paper_1704_03116_b200 as dope
from paper_1704_03116_b200 import compare
from paper_1704_03116_b200 import workloads as W


def test_metrics():
    a = np.array([1, 1, 0, 0]); b = np.array([1, 0, 0, 0])
    assert compare.dice(a, b) == pytest.approx(2 / 3)
    assert compare.dice(np.zeros(3), np.zeros(3)) == 1.0
    assert compare.relative_energy_diff(-100.0, -99.0) == pytest.approx(1.0)


def _oracle_cut(model):
    import oracle as orc
    w = model.weights
    lab, flow = orc.bk_maxflow(model.unary.copy(), w.rows.astype(np.int32), w.cols.astype(np.int32),
                               model.lam * w.vals, model.lam * w.vals)
    return np.asarray(lab, dtype=np.int8), flow


def _model(wl):
    rows, cols, vals = wl.pair_arrays()
    return dope.EnergyModel(np.asarray(wl.u, dtype=np.float64), dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)


@pytest.mark.gpu
@pytest.mark.parametrize("size,seed", [(64, 1), (256, 2), (512, 3)])
def test_grid_cut_integer_matches_bk(size, seed):
    wl = W.mini_disks(size, 32, 6, 2, 1, seed=seed, rmax=size / 4)
    model = _model(wl)
    lab, flow = compare.solve_binary_grid(model.unary, model.weights, model.lam, wl.dims)
    ref, rflow = _oracle_cut(model)
    assert np.array_equal(lab, ref)
    assert flow == pytest.approx(rflow, rel=1e-12, abs=1e-9)


@pytest.mark.gpu
def test_grid_cut_float_8conn_within_tolerance():
    wl = W.c2(size=128, block=32, iters=1)
    model = _model(wl)
    lab, _ = compare.solve_binary_grid(model.unary, model.weights, model.lam, wl.dims)
    ref, _ = _oracle_cut(model)
    assert np.count_nonzero(lab != ref) <= 1e-4 * lab.size
    e = dope.evaluate_energy(model, lab.astype(float))
    er = dope.evaluate_energy(model, ref.astype(float))
    assert abs(e - er) <= 1e-6 * abs(er)


@pytest.mark.gpu
def test_run_serial_compare_mode():
    wl = W.mini_disks(256, 64, 6, 2, 1, seed=4, rmax=60.0)
    model = _model(wl)
    shape = dope.GridShape(wl.dims)
    serial, e_serial, _ = compare.run_serial(model, shape)
    part = dope.make_partition(shape, wl.kpa, 0)
    dist, state = dope.run(model, part, dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=40))
    e_dist = dope.evaluate_energy(model, dist.astype(float))
    assert e_serial <= e_dist + 1e-9                 # the serial cut is the global optimum
    assert compare.dice(serial, dist) > 0.9
    assert abs(compare.relative_energy_diff(e_serial, e_dist)) < 5.0
