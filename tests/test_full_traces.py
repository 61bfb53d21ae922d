"""Full-length parity on every BASELINE config at full size, every iteration.

The fixtures (tests/golden/full_*.npz, made by tests/golden/make_fulltrace.py)
hold the CPU oracle's run of each config -- the oracle is itself pinned
bit-for-bit to traces the reference produced (tests/test_oracle_golden.py).
Each GPU run goes through the public `run()` in audit mode
(AdmmConfig.digests): after every iteration the device adds the iteration's
state digest -- order-independent position-weighted sums of the block labels
yhat, 2y and the multipliers a (dope_oracle.c state_digest) -- so the whole
trajectory is compared without copying 100 x 16.7 M labels to the host.

Integer configs (C1, C3, C4, C5 b16-b128): bit-exact -- every iteration's
energy, max block residual, clamp flag and (yhat, y, a) digest, the
iteration count / best iterate, the returned state.y, labels and
multipliers.  residual_sq: rtol 1e-12 (numpy's summation order in the oracle).
Float config C2: BASELINE's bar -- energies within 1e-5 relative (every
iteration and final), <= 0.01 % label disagreement.
"""
import numpy as np
import pytest

import paper_1704_03116_b200 as dope
from paper_1704_03116_b200 import workloads as W
from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

INT_CONFIGS = ["C1", "C3", "C4", "C5-B16", "C5-B32", "C5-B64", "C5-B128"]


def _fixture(name):
    return load_golden(f"full_{name.lower()}.npz")


def _model(wl):
    rows, cols, vals = wl.pair_arrays()
    u = wl.u.astype(np.float64)
    model = dope.EnergyModel(u, dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    return model, part


def _u_checksum(u):
    import oracle as orc
    z = np.zeros(u.size, dtype=np.uint8)
    if np.all(u == np.round(u)):
        return orc.state_digest(z, u.astype(np.float64) / 2.0, np.zeros(u.size))[1]
    return np.uint64(int(np.ascontiguousarray(u, dtype=np.float64).view(np.int64)
                         .astype(np.uint64).sum(dtype=np.uint64)))


def _digest(yhat, y, a):
    import oracle as orc
    return orc.state_digest(yhat, y, a)


@pytest.mark.parametrize("name", INT_CONFIGS)
def test_integer_config_full_run_bit_exact_every_iteration(name):
    g = _fixture(name)
    wl = W.by_name(name)
    assert _u_checksum(wl.u) == g["u_checksum"], "workload generator differs from the fixture's"
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=wl.iters, digests=True)
    labels, state = dope.run(model, part, cfg)
    it = int(g["iterations"])
    assert state.iteration == it
    assert state.converged == bool(g["converged"])
    assert state.best_iteration == int(g["best_iteration"])
    assert np.array_equal([t.energy for t in state.trace], g["energy"])
    assert np.array_equal([t.max_block_residual for t in state.trace], g["max_block_residual"])
    assert np.array_equal([t.clamped for t in state.trace], g["clamped"])
    np.testing.assert_allclose([t.residual_sq for t in state.trace], g["residual_sq"], rtol=1e-12)
    bad = [t + 1 for t in range(it) if not np.array_equal(state.digests[t], g["digests"][t])]
    assert not bad, f"state digests differ at iterations {bad[:10]}"
    fin = _digest(state.labels_global().astype(np.uint8), state.y, state.multipliers_global())
    assert np.array_equal(fin, g["final_digest"])
    assert _digest(labels.astype(np.uint8), np.zeros(wl.n), np.zeros(wl.n))[0] == g["labels_digest"]


def test_float_config_c2_full_run_within_baseline_tolerance():
    g = _fixture("C2")
    wl = W.by_name("C2")
    assert _u_checksum(wl.u) == g["u_checksum"]
    model, part = _model(wl)
    cfg = dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=wl.iters, digests=True)
    labels, state = dope.run(model, part, cfg)
    assert state.iteration == int(g["iterations"])
    e = np.array([t.energy for t in state.trace])
    np.testing.assert_allclose(e, g["energy"], rtol=1e-5)
    assert abs(e[-1] - g["energy"][-1]) <= 1e-5 * abs(g["energy"][-1])
    ref_labels = np.unpackbits(g["labels_bits"])[:wl.n]
    assert np.mean(labels != ref_labels) <= 1e-4
    ref_yhat = np.unpackbits(g["yhat_bits"])[:wl.n]
    assert np.mean(state.labels_global() != ref_yhat) <= 1e-4
    same = int(sum(int(state.digests[t][0]) == int(g["digests"][t][0]) for t in range(state.iteration)))
    print(f"C2: block labels identical to the oracle's in {same}/{state.iteration} iterations")


def test_fixtures_present():
    for name in INT_CONFIGS + ["C2"]:
        assert (GOLDEN / f"full_{name.lower()}.npz").exists(), name
