"""Host-side API pieces that need no GPU: containers, geometry, partitions,
state semantics, the sharded path's refusals (CPU only)."""
import numpy as np
import pytest

import paper_1704_03116_b200 as dope
from paper_1704_03116_b200 import sharded, workloads as W
from paper_1704_03116_b200.partition import axis_ranges, box_pixels


def test_sparse_weights_canonical_form_and_csr_views(rng):
    w = dope.SparseWeights(5, [3, 0, 4], [1, 2, 2], [1.5, 2.0, 0.25])
    assert w.rows.tolist() == [1, 0, 2] and w.cols.tolist() == [3, 2, 4]
    m = w.to_csr().toarray()
    assert np.array_equal(m, m.T) and m[1, 3] == 1.5 and m[4, 2] == 0.25
    indptr, indices, data = w.adjacency()
    assert indptr.tolist() == [0, 1, 2, 4, 5, 6]
    lap = w.laplacian().toarray()
    assert np.allclose(lap.sum(axis=1), 0.0) and np.allclose(np.diag(lap), w.degrees())
    back = dope.SparseWeights.from_symmetric(m)
    assert sorted(zip(back.rows, back.cols, back.vals)) == sorted(zip(w.rows, w.cols, w.vals))
    with pytest.raises(ValueError):
        dope.SparseWeights.from_symmetric(np.array([[0, 1.0], [2.0, 0]]))
    with pytest.raises(dope.NonSubmodularError):
        dope.SparseWeights(2, [0], [1], [-1.0])
    with pytest.raises(ValueError):
        dope.SparseWeights(2, [1], [1], [1.0])


def test_grid_indexing_round_trip():
    shape = dope.GridShape((3, 4, 5))
    assert shape.strides == (20, 5, 1) and shape.n == 60
    for g in (0, 7, 59):
        assert dope.index_of(shape, dope.coords_of(shape, g)) == g
    with pytest.raises(ValueError):
        dope.GridShape((4,))


def test_partition_rules():
    assert axis_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert axis_ranges(10, 3, 25) == [(0, 5), (3, 8), (6, 10)]
    p = dope.make_partition(dope.GridShape((5, 4)), (2, 2), 25)
    assert p.counts.max() == 4 and p.blocks[3].extent == ((2, 5), (1, 4))
    assert np.array_equal(p.blocks[1].pixels, box_pixels(p.shape, ((0, 4), (1, 4))))
    lazy = dope.make_partition(dope.GridShape((64, 64)), (4, 4), 0, materialize=False)
    assert lazy.blocks[5].size == 256 and lazy.blocks[5].pixels.size == 0


def test_state_semantics_on_the_host():
    part = dope.make_partition(dope.GridShape((3, 3)), (1, 1), 0)
    st = dope.init_state(part, 4.0)
    assert np.all(st.y == 0.5) and st.mu == 4.0 and st.block_labels[0].dtype == np.int8
    st.multipliers[0] += 2.0          # a plain list of arrays: edits stick
    assert np.all(st.multipliers[0] == 2.0)
    assert dope.binarize(np.array([0.49, 0.5, 0.51])).tolist() == [0, 1, 1]


def test_sharded_path_refuses_what_it_cannot_run_exactly():
    wl = W.mini_disks(256, 64, 8, 2, 5, seed=1)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u.astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    for cfg in (dope.AdmmConfig(mu0=1.0, max_iters=5),                  # mu_fact 1.05
                dope.AdmmConfig(mu0=1.5, mu_fact=1.0, max_iters=5),     # non-integer mu
                dope.AdmmConfig(mu0=3.0, mu_fact=1.0, max_iters=5)):    # 3 does not divide lam*w
        with pytest.raises(NotImplementedError):
            sharded.shard_for_rank(model, part, cfg, 0, 1)
