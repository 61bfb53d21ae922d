"""The general-path oracle (oracle/general.py) pinned against the reference's
own fixtures (tests/golden/gen_*.npz): overlapping partitions and the
reference's growing-mu schedule.  CPU only."""
import numpy as np
import pytest

from conftest import load_golden

CASES = ["c2ov25", "c2ov25_long", "int_ov10", "mufact", "mufact_long"]


def spec_from(g):
    import general as og
    dims = tuple(int(d) for d in g["dims"])
    n = dims[0] * dims[1]
    wp = g["wplanes"]
    planes = [np.full(n, float(w)) for w in wp] if wp.ndim == 1 else [np.asarray(w) for w in wp]
    planes = planes + [np.zeros(n)] * (4 - len(planes))
    if wp.ndim == 1:   # constant weights: zero the pairs that leave the grid
        H, W = dims
        E = planes[0].reshape(H, W).copy(); E[:, -1] = 0
        S = planes[1].reshape(H, W).copy(); S[-1, :] = 0
        planes[0], planes[1] = E.ravel(), S.ravel()
    kpa = tuple(d // int(b) for d, b in zip(dims, g["block"]))
    return og.GeneralSpec(dims, int(g["conn"]), g["u"], planes, float(g["lam"]), kpa, int(g["overlap"]))


@pytest.mark.parametrize("case", CASES)
def test_general_oracle_matches_reference(case):
    import general as og
    g = load_golden(f"gen_{case}.npz")
    spec = spec_from(g)
    assert np.array_equal(spec.q.ravel().astype(np.int64), g["counts"])
    out = og.run(spec, float(g["mu0"]), float(g["mu_fact"]), float(g["eps"]), int(g["max_iters"]))
    assert out["iterations"] == int(g["iterations"])
    assert out["converged"] == bool(g["converged"])
    assert out["best_iteration"] == int(g["best_iteration"])
    np.testing.assert_allclose(out["energy"], g["energy"], rtol=1e-10)
    np.testing.assert_allclose(out["mu"], g["mu"], rtol=1e-14)
    np.testing.assert_allclose(out["max_block_residual"], g["max_block_residual"], rtol=1e-9, atol=1e-12)
    assert np.array_equal(out["labels"], g["labels"])
    np.testing.assert_allclose(out["y"], g["y"], atol=1e-9)
    np.testing.assert_allclose(out["a_copies"], g["a_copies"], atol=1e-9)
    hist = np.unpackbits(g["yhat_bits"], axis=1)[:, :out["yhat_copies"].size]
    assert np.array_equal(out["yhat_copies"].astype(np.uint8), hist[-1])
