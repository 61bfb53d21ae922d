"""The general graph path (csrc/dope_gstep.cu + batched block min cuts) against
runs of the reference itself (tests/golden/graph_*.npz, made by
tests/golden/make_golden.py --only-graph): models and partitions the lattice
kernels do not take -- 3D overlapping partitions with q up to 8, the
reference's default 3D config, kernel-5 / 18-connected windows.

Integer models with power-of-two block counts: every value is a dyadic
rational, so the float64 device arithmetic is exact -- bit-exact every
iteration (energies, max residuals, clamp flags, every block copy's labels),
final y, labels and multiplier copies.  Float models: energies within 1e-9
relative every iteration, identical block labels.
"""
import numpy as np
import pytest

import paper_1704_03116_b200 as dope
from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

CASES = sorted(p.name[len("graph_"):-len(".npz")] for p in GOLDEN.glob("graph_*.npz"))


def _setup(g):
    dims = tuple(int(d) for d in g["dims"])
    w = dope.SparseWeights(int(np.prod(dims)), g["rows"], g["cols"], g["vals"])
    model = dope.EnergyModel(g["u"], w, float(g["lam"]))
    part = dope.make_partition(dope.GridShape(dims), tuple(int(k) for k in g["kpa"]), int(g["overlap"]))
    mu0 = None if np.isnan(g["cfg_mu0"]) else float(g["cfg_mu0"])
    eps = None if np.isnan(g["cfg_eps"]) else float(g["cfg_eps"])
    cfg = dope.AdmmConfig(mu0=mu0, mu_fact=float(g["cfg_mu_fact"]), eps=eps, max_iters=int(g["max_iters"]))
    return model, part, cfg


@pytest.mark.parametrize("case", CASES)
def test_run_matches_reference(case):
    g = load_golden(f"graph_{case}.npz")
    model, part, cfg = _setup(g)
    labels, state = dope.run(model, part, cfg)
    assert state.iteration == int(g["iterations"])
    assert state.converged == bool(g["converged"])
    assert state.best_iteration == int(g["best_iteration"])
    assert np.array_equal([t.clamped for t in state.trace], g["clamped"])
    np.testing.assert_allclose([t.mu for t in state.trace], g["mu"], rtol=1e-15)
    hist = np.unpackbits(g["yhat_bits"], axis=1)[:, :sum(b.size for b in part.blocks)]
    copies = np.concatenate(state.block_labels).astype(np.uint8)
    assert np.array_equal(copies, hist[state.iteration - 1])
    e = np.array([t.energy for t in state.trace])
    if bool(g["integer"]):
        assert np.array_equal(e, g["energy"])
        assert np.array_equal([t.max_block_residual for t in state.trace], g["max_block_residual"])
        np.testing.assert_allclose([t.residual_sq for t in state.trace], g["residual_sq"], rtol=1e-12)
        assert np.array_equal(state.y, g["y"])
        assert np.array_equal(np.concatenate(state.multipliers), g["a_copies"])
    else:
        np.testing.assert_allclose(e, g["energy"], rtol=1e-9)
        np.testing.assert_allclose(state.y, g["y"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(np.concatenate(state.multipliers), g["a_copies"], rtol=1e-9, atol=1e-9)
    assert np.array_equal(labels, g["labels"])


@pytest.mark.parametrize("case", ["int3d_ov25", "k5_sched"])
def test_step_api_reproduces_the_run(case):
    """init_state -> update_blocks -> update_global -> block_residuals ->
    evaluate_energy -> update_multipliers, through the public step functions,
    every iteration's block labels against the reference's trace."""
    g = load_golden(f"graph_{case}.npz")
    model, part, cfg = _setup(g)
    problems = dope.assemble_block_problems(model, part)
    state = dope.init_state(part, cfg.resolved_mu0(part.shape.ndim))
    hist = np.unpackbits(g["yhat_bits"], axis=1)[:, :sum(b.size for b in part.blocks)]
    for it in range(int(g["iterations"])):
        dope.update_blocks(state, problems, model.lam, cfg)
        assert np.array_equal(np.concatenate(state.block_labels).astype(np.uint8), hist[it]), it
        dope.update_global(state, problems, part, model.lam)
        assert state.clamped_last == bool(g["clamped"][it])
        res = dope.block_residuals(state, part)
        e = dope.evaluate_energy(model, state.y)
        if bool(g["integer"]):
            assert e == g["energy"][it] and float(res.max()) == g["max_block_residual"][it]
        else:
            assert e == pytest.approx(g["energy"][it], rel=1e-9)
        dope.update_multipliers(state, part, cfg.mu_fact)
