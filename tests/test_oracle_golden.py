"""Pin the CPU oracle against the reference's own outputs (tests/golden/).

The oracle restates _core.pyx (BK) and admm.run on q == 1 lattices; these
tests show it reproduces the reference bit-for-bit on every committed
fixture before it is trusted as the GPU checker.
"""
import numpy as np
import pytest

import oracle as orc
from conftest import golden_cases, load_golden, spec_from_golden


def test_bk_restatement_matches_reference_outputs():
    g = load_golden("bk_graphs.npz")
    mo, po = g["m_off"], g["p_off"]
    for k in range(len(mo) - 1):
        sl_m, sl_p = slice(mo[k], mo[k + 1]), slice(po[k], po[k + 1])
        lab, flow = orc.bk_maxflow(g["tcap"][sl_m], g["pi"][sl_p], g["pj"][sl_p],
                                   g["cij"][sl_p], g["cji"][sl_p])
        assert np.array_equal(lab, g["labels"][sl_m]), k
        assert flow == g["flows"][k], k          # bit-identical arithmetic


def test_bk_restatement_matches_compiled_reference_core(rng):
    core = orc.reference_core()
    if core is None:
        pytest.skip("oracle/_ref not built")
    for _ in range(100):
        m = int(rng.integers(1, 50))
        pairs = [(i, j) for i in range(m) for j in range(i + 1, m) if rng.random() < 0.2]
        pi = np.array([p[0] for p in pairs], dtype=np.int32)
        pj = np.array([p[1] for p in pairs], dtype=np.int32)
        cij, cji = rng.random(pi.size) * 3, rng.random(pi.size) * 3
        tcap = rng.uniform(-4, 4, m)
        if rng.random() < 0.5:
            tcap = np.round(tcap)
        a = core.bk_maxflow(tcap.copy(), pi, pj, cij, cji)
        b = orc.bk_maxflow(tcap, pi, pj, cij, cji)
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]


def test_bk_edge_cases():
    lab, flow = orc.bk_maxflow(np.zeros(0), [], [], [], [])
    assert lab.size == 0 and flow == 0.0
    lab, _ = orc.bk_maxflow(np.array([2.0, -1.0, 0.0, -0.5]), [], [], [], [])
    assert lab.tolist() == [0, 1, 0, 1]          # ties prefer 0 (test_maxflow.py:51-54)
    lab, flow = orc.bk_maxflow(np.array([4.0, -4.0]), [0], [1], [1.0], [10.0])
    assert lab.tolist() == [0, 1] and flow == 1.0  # asymmetric caps (test_maxflow.py:184-192)


@pytest.mark.parametrize("case", golden_cases())
def test_oracle_run_matches_reference_trace(case):
    g = load_golden(f"run_{case}.npz")
    spec = spec_from_golden(g)
    out = orc.run(spec, float(g["rho"]), 1.0, 0.0, int(g["max_iters"]), threads=2,
                  keep_history=True)
    assert out["iterations"] == int(g["iterations"])
    assert out["converged"] == bool(g["converged"])
    assert out["best_iteration"] == int(g["best_iteration"])
    hist = np.unpackbits(g["yhat_bits"], axis=1)[:, :spec.n]
    assert np.array_equal(out["yhat_history"], hist)
    assert np.array_equal(out["clamped"], g["clamped"])
    assert np.array_equal(out["mu"], g["mu"])
    assert np.array_equal(out["labels"], g["labels"])
    if "wplanes" in g:   # float config: the reference's BLAS dot order is not restated
        np.testing.assert_allclose(out["energy"], g["energy"], rtol=1e-13)
        np.testing.assert_allclose(out["max_block_residual"], g["max_block_residual"], rtol=1e-13)
        np.testing.assert_allclose(out["residual_sq"], g["residual_sq"], rtol=1e-12)
        np.testing.assert_allclose(out["y"], g["y"], atol=1e-12)
        np.testing.assert_allclose(out["a"], g["a"], atol=1e-12)
    else:                # integer configs: bit-exact
        assert np.array_equal(out["energy"], g["energy"])
        assert np.array_equal(out["max_block_residual"], g["max_block_residual"])
        np.testing.assert_allclose(out["residual_sq"], g["residual_sq"], rtol=1e-12)
        assert np.array_equal(out["y"], g["y"])
        assert np.array_equal(out["a"], g["a"])
