"""General path vs the reference: overlapping partitions
(overlap_pct 10 / 25, q in {1, 2, 4}) and the reference's default growing mu.

Fixtures gen_*.npz are admm.run outputs of the reference itself
(tests/golden/make_golden.py, main_general).  Float parity bar (BASELINE):
final energy within 1e-5 relative and <= 0.01 % label disagreement; we also
hold every iteration's energy and mu, the stop iteration and the per-copy
multipliers to tight tolerances.
"""
import numpy as np
import pytest

import paper_1704_03116_b200 as dope
from paper_1704_03116_b200 import workloads as W
from conftest import load_golden

pytestmark = pytest.mark.gpu

CASES = ["c2ov25", "c2ov25_long", "int_ov10", "mufact", "mufact_long"]


def _model(g):
    dims = tuple(int(d) for d in g["dims"])
    conn = int(g["conn"])
    wp = g["wplanes"]
    weights = [float(w) for w in wp] if wp.ndim == 1 else [np.asarray(w) for w in wp]
    wl = W.Workload("g", dims, tuple(int(b) for b in g["block"]), conn, g["u"], weights,
                    float(g["lam"]), 1.0, int(g["max_iters"]), wp.ndim == 1)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(np.asarray(g["u"], dtype=np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             float(g["lam"]))
    part = dope.make_partition(dope.GridShape(dims), wl.kpa, int(g["overlap"]))
    cfg = dope.AdmmConfig(mu0=float(g["mu0"]), mu_fact=float(g["mu_fact"]), eps=float(g["eps"]),
                          max_iters=int(g["max_iters"]))
    return model, part, cfg


@pytest.mark.parametrize("case", CASES)
def test_general_matches_reference(case):
    g = load_golden(f"gen_{case}.npz")
    model, part, cfg = _model(g)
    if int(g["overlap"]):
        assert int(part.counts.max()) > 1
    labels, state = dope.run(model, part, cfg)
    it = int(g["iterations"])
    assert state.iteration == it
    assert state.converged == bool(g["converged"])
    e = np.array([t.energy for t in state.trace])
    np.testing.assert_allclose(e, g["energy"], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose([t.mu for t in state.trace], g["mu"], rtol=1e-12)
    np.testing.assert_allclose([t.max_block_residual for t in state.trace], g["max_block_residual"],
                               rtol=1e-6, atol=1e-9)
    assert abs(e[-1] - g["energy"][-1]) <= 1e-5 * abs(g["energy"][-1])
    assert state.best_iteration == int(g["best_iteration"])
    dis = np.count_nonzero(labels != g["labels"])
    assert dis <= 1e-4 * labels.size, dis
    np.testing.assert_allclose(state.y, g["y"], atol=1e-6)
    a = np.concatenate(state.multipliers)
    np.testing.assert_allclose(a, g["a_copies"], atol=1e-6)
    # per-iteration block labels (every copy)
    hist = np.unpackbits(g["yhat_bits"], axis=1)[:, :a.size]
    assert np.array_equal(np.concatenate(state.block_labels).astype(np.uint8), hist[it - 1])


def test_general_graph_and_eager_agree():
    g = load_golden("gen_int_ov10.npz")
    model, part, cfg = _model(g)
    l1, s1 = dope.run(model, part, cfg)
    cfg.use_graph = False
    l2, s2 = dope.run(model, part, cfg)
    assert np.array_equal(l1, l2)
    assert [t.energy for t in s1.trace] == [t.energy for t in s2.trace]


@pytest.mark.parametrize("overlap,conn", [(25, 8), (10, 4)])
def test_general_vs_oracle_256(overlap, conn):
    """256^2, 8x8 blocks of 32 grown by the overlap, growing mu: B200 vs the
    general-path oracle (itself pinned to the reference's fixtures)."""
    import general as og
    if conn == 8:
        wl = W.c2(size=256, block=32, iters=12)
    else:
        wl = W.mini_disks(256, 32, 8, 2, 12, seed=11, rmax=60.0)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(np.asarray(wl.u, dtype=np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, overlap)
    cfg = dope.AdmmConfig(mu0=2.0, mu_fact=1.05, eps=0.0, max_iters=12)
    labels, state = dope.run(model, part, cfg)
    from paper_1704_03116_b200.lowering import lattice_planes
    planes, c = lattice_planes(model, wl.dims)
    assert c == conn
    spec = og.GeneralSpec(wl.dims, conn, wl.u, planes, wl.lam, wl.kpa, overlap)
    ref = og.run(spec, 2.0, 1.05, 0.0, 12)
    assert state.iteration == ref["iterations"]
    np.testing.assert_allclose([t.energy for t in state.trace], ref["energy"], rtol=1e-6)
    assert np.count_nonzero(labels != ref["labels"]) <= 1e-4 * labels.size


def test_default_config_on_integer_model_uses_general_path():
    """mu0 = 100 with mu_fact = 1 does not divide lambda*w: run() takes the
    general path and still matches the general oracle."""
    import general as og
    wl = W.mini_disks(128, 32, 6, 2, 10, seed=12, rmax=40.0)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(np.asarray(wl.u, dtype=np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0)
    cfg = dope.AdmmConfig(mu0=None, mu_fact=1.0, eps=0.0, max_iters=10)
    labels, state = dope.run(model, part, cfg)
    from paper_1704_03116_b200.lowering import lattice_planes
    planes, c = lattice_planes(model, wl.dims)
    ref = og.run(og.GeneralSpec(wl.dims, c, wl.u, planes, wl.lam, wl.kpa, 0), 100.0, 1.0, 0.0, 10)
    np.testing.assert_allclose([t.energy for t in state.trace], ref["energy"], rtol=1e-6)
    assert np.array_equal(labels, ref["labels"])
