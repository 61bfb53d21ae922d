"""Model construction vs the reference's own builders
(tests/golden/inputs_*.npz, made by tests/golden/make_golden.py)."""
import numpy as np
import pytest

import paper_1704_03116_b200 as dope
from paper_1704_03116_b200 import inputs as din
from conftest import load_golden


def _img2d(g):
    return din.GridImage(dope.GridShape(tuple(int(d) for d in g["dims"])), g["data"], g["seeds"])


def test_half_kernel_offsets():
    assert len(din.half_kernel_offsets(2, 3)) == 4 and len(din.half_kernel_offsets(2, 9)) == 40
    assert len(din.half_kernel_offsets(3, 3)) == 9
    assert all(o > (0, 0, 0) for o in din.half_kernel_offsets(3, 9))


def test_color_model_matches_reference():
    g = load_golden("inputs_2d.npz")
    cm = din.fit_color_model(_img2d(g), rng=np.random.default_rng(0))
    np.testing.assert_array_equal(cm.fg_centroids, g["fg_c"])
    np.testing.assert_array_equal(cm.bg_centroids, g["bg_c"])
    np.testing.assert_array_equal(cm.fg_weights, g["fg_w"])
    np.testing.assert_array_equal(cm.bg_weights, g["bg_w"])
    assert cm.bandwidth == float(g["bw"])


@pytest.mark.gpu
@pytest.mark.parametrize("fixture", ["inputs_2d.npz", "inputs_3d.npz"])
@pytest.mark.parametrize("k", [3, 5])
def test_potts_weights_and_sigma_on_gpu(fixture, k):
    g = load_golden(fixture)
    shape = dope.GridShape(tuple(int(d) for d in g["dims"]))
    img = din.GridImage(shape, g["data"])
    s = din.estimate_sigma(img, k)
    assert s == pytest.approx(float(g[f"sigma{k}"]), rel=1e-12)
    w = din.build_potts_weights(img, k, float(g[f"sigma{k}"]), contrast=True)
    np.testing.assert_array_equal(w.rows, g[f"rows{k}"])
    np.testing.assert_array_equal(w.cols, g[f"cols{k}"])
    np.testing.assert_allclose(w.vals, g[f"vals{k}"], rtol=1e-13, atol=0)


@pytest.mark.gpu
def test_unaries_on_gpu():
    g = load_golden("inputs_2d.npz")
    img = _img2d(g)
    cm = din.ColorModel(g["fg_c"], g["bg_c"], g["fg_w"], g["bg_w"], float(g["bw"]))
    u = din.compute_unaries(img, cm)
    np.testing.assert_allclose(u, g["u"], rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_built_model_runs():
    """GPU-built weights / unaries feed the general path end to end."""
    g = load_golden("inputs_2d.npz")
    img = _img2d(g)
    cm = din.fit_color_model(img, rng=np.random.default_rng(0))
    u = din.compute_unaries(img, cm)
    w = din.build_potts_weights(img, 3, din.estimate_sigma(img, 3))
    model = dope.EnergyModel(np.clip(u, -50, 50), w, 1.0)
    part = dope.make_partition(img.shape, (3, 4), 25)
    labels, state = dope.run(model, part, dope.AdmmConfig(max_iters=20))
    assert labels.shape == (img.shape.n,) and state.iteration >= 1
    assert np.isfinite([t.energy for t in state.trace]).all()
