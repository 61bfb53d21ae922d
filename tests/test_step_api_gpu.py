"""The reference's step-level API on the device (admm.py:113-204,
blockform.py:89-105, solvers.py:111-147), checked the way the reference's own
tests check it (pkg/tests/test_admm.py:60-192, test_blockform.py): against a
dense restatement of the block operators (tests/dense_oracle.py), finite
differences, enumeration, and the behaviours the reference pins (rounding
under a huge penalty, exact halves resolving to 0, block means without
coupling, multiplier accumulation, BlockSolveError carrying the block id).
Models are random 8-connected windows on small grids with random partitions
(overlap 0 / 10 / 25) -- the general graph path.
"""
import numpy as np
import pytest

import paper_1704_03116_b200 as dope
from dense_oracle import DenseOps

pytestmark = pytest.mark.gpu


def window_pairs(dims):
    """Every 8-connected neighbour pair (3x3 window) of a 2D grid, i < j."""
    H, W = dims
    idx = np.arange(H * W).reshape(H, W)
    rows, cols = [], []
    for dy, dx in ((0, 1), (1, -1), (1, 0), (1, 1)):
        a = idx[max(0, -dy):H - max(0, dy), max(0, -dx):W - max(0, dx)]
        b = idx[max(0, dy):H + min(0, dy), max(0, dx):W + min(0, dx)]
        rows.append(a.ravel())
        cols.append(b.ravel())
    return np.concatenate(rows), np.concatenate(cols)


def random_model(rng, dims, lam_max=2.0, scale=5.0):
    r, c = window_pairs(dims)
    n = int(np.prod(dims))
    w = dope.SparseWeights(n, r, c, rng.random(r.size) + 0.05)
    return dope.EnergyModel(rng.uniform(-scale, scale, n), w, float(rng.uniform(0.0, lam_max)))


def random_case(rng):
    dims = (int(rng.integers(2, 8)), int(rng.integers(2, 8)))
    model = random_model(rng, dims)
    kpa = tuple(int(rng.integers(1, max(2, d // 2 + 1))) for d in dims)
    part = dope.make_partition(dope.GridShape(dims), kpa, int(rng.choice([0, 10, 25])))
    return model, part


def random_state(rng, part):
    yhat = [rng.integers(0, 2, b.size).astype(np.int8) for b in part.blocks]
    mults = [rng.normal(0, 0.5, b.size) for b in part.blocks]
    return yhat, mults


def test_solve_global_matches_dense_oracle(rng):
    for _ in range(12):
        model, part = random_case(rng)
        problems = dope.assemble_block_problems(model, part)
        yhat, mults = random_state(rng, part)
        mu = float(rng.uniform(1, 50))
        y = dope.solve_global(problems, part, yhat, mults, mu, model.lam)
        ref = DenseOps(model, part).solve_global(yhat, mults, mu, model.lam)
        np.testing.assert_allclose(y, ref, atol=1e-10)


def test_block_objective_and_views_match_dense_oracle(rng):
    for _ in range(8):
        model, part = random_case(rng)
        problems = dope.assemble_block_problems(model, part)
        ops = DenseOps(model, part)
        y = rng.random(model.n)
        mu = float(rng.uniform(0, 20))
        for k, bp in enumerate(problems):
            a = rng.normal(size=bp.size)
            lin, pw, scale = dope.block_objective(bp, y, a, mu, model.lam)
            np.testing.assert_allclose(lin, ops.linear(k, y, a, mu, model.lam), atol=1e-10)
            assert scale == model.lam
            np.testing.assert_allclose(bp.r_diag, ops.r[k], atol=1e-12)
            np.testing.assert_allclose(bp.c_rows.toarray(), ops.C[k], atol=1e-12)
            dense_w = np.zeros((bp.size, bp.size))
            dense_w[pw.rows, pw.cols] = pw.vals
            np.testing.assert_allclose(dense_w + dense_w.T, ops.What[k], atol=1e-12)
            np.testing.assert_allclose(bp.u_hat, model.unary[bp.block.pixels] / ops.q[bp.block.pixels])


def test_solve_global_zeroes_the_consensus_gradient(rng):
    for _ in range(8):
        model, part = random_case(rng)
        problems = dope.assemble_block_problems(model, part)
        yhat, mults = random_state(rng, part)
        mu = float(rng.uniform(1, 100))
        y = dope.solve_global(problems, part, yhat, mults, mu, model.lam)
        ops = DenseOps(model, part)
        assert dope.consensus_objective(problems, part, yhat, mults, mu, model.lam, y) == pytest.approx(
            ops.objective(yhat, mults, mu, model.lam, y), rel=1e-12, abs=1e-12)
        h = 1e-5
        for c in rng.integers(0, model.n, size=min(6, model.n)):
            yp, ym = y.copy(), y.copy()
            yp[c] += h
            ym[c] -= h
            g = (dope.consensus_objective(problems, part, yhat, mults, mu, model.lam, yp)
                 - dope.consensus_objective(problems, part, yhat, mults, mu, model.lam, ym)) / (2 * h)
            assert abs(g) <= 1e-6 * (1 + mu * part.counts.max())


@pytest.mark.parametrize("solver", [dope.MAXFLOW, dope.EXHAUSTIVE])
def test_update_blocks_rounds_under_a_huge_penalty(rng, solver):
    shape = dope.GridShape((4, 4))
    model = random_model(rng, shape.dims, lam_max=0.5, scale=1.0)
    part = dope.make_partition(shape, (2, 2), 0)
    problems = dope.assemble_block_problems(model, part)
    state = dope.init_state(part, mu0=1e9)
    state.y = rng.random(shape.n)
    dope.update_blocks(state, problems, model.lam, dope.AdmmConfig(solver=solver))
    for b, lab in zip(part.blocks, state.block_labels):
        assert np.array_equal(lab, (state.y[b.pixels] > 0.5).astype(np.int8))


def test_exact_half_resolves_to_zero():
    model = dope.EnergyModel(np.zeros(4), dope.SparseWeights(4, [0], [1], [1.0]), lam=0.0)
    part = dope.make_partition(dope.GridShape((2, 2)), (1, 1), 0)
    problems = dope.assemble_block_problems(model, part)
    for solver in (dope.MAXFLOW, dope.EXHAUSTIVE):
        state = dope.init_state(part, mu0=1e9)
        dope.update_blocks(state, problems, model.lam, dope.AdmmConfig(solver=solver))
        assert state.block_labels[0].tolist() == [0, 0, 0, 0]


def test_disjoint_blocks_solve_standalone(rng):
    w = dope.SparseWeights(8, [0, 1, 2, 6], [4, 5, 3, 7], [1.0, 0.5, 2.0, 1.5])
    model = dope.EnergyModel(rng.normal(size=8), w, lam=1.0)
    part = dope.make_partition(dope.GridShape((2, 4)), (1, 2), 0)
    problems = dope.assemble_block_problems(model, part)
    state = dope.init_state(part, mu0=1.0)
    state.mu = 0.0
    dope.update_blocks(state, problems, model.lam, dope.AdmmConfig(solver=dope.MAXFLOW))
    for bp, lab in zip(problems, state.block_labels):
        expected, _ = dope.exhaustive_minimize(model.unary[bp.block.pixels], bp.w_hat, model.lam)
        assert np.array_equal(lab, expected)


def test_update_global_is_the_block_mean_without_coupling(rng):
    model = dope.EnergyModel(rng.normal(size=36), dope.SparseWeights(36, [0], [1], [1.0]), lam=0.0)
    part = dope.make_partition(dope.GridShape((6, 6)), (2, 2), 25)
    problems = dope.assemble_block_problems(model, part)
    state = dope.init_state(part, mu0=50.0)
    state.block_labels = [rng.integers(0, 2, b.size).astype(np.int8) for b in part.blocks]
    dope.update_global(state, problems, part, model.lam)
    acc = np.zeros(36)
    for b, lab in zip(part.blocks, state.block_labels):
        acc[b.pixels] += lab
    np.testing.assert_allclose(state.y, acc / part.counts)


def test_solve_global_affine_shift_and_positive_mu(rng):
    model = dope.EnergyModel(rng.normal(size=9), dope.SparseWeights(9, [0], [1], [1.0]), lam=0.0)
    part = dope.make_partition(dope.GridShape((3, 3)), (1, 1), 0)
    problems = dope.assemble_block_problems(model, part)
    yhat = [rng.integers(0, 2, 9).astype(float)]
    y = dope.solve_global(problems, part, yhat, [np.full(9, 0.3)], 10.0, model.lam)
    np.testing.assert_allclose(y, yhat[0] + 0.3)
    with pytest.raises(ValueError):
        dope.solve_global(problems, part, [np.zeros(9)], [np.zeros(9)], 0.0, 1.0)


def test_update_multipliers_fixed_point_accumulation_and_mu_schedule():
    part = dope.make_partition(dope.GridShape((2, 2)), (1, 1), 0)
    state = dope.init_state(part, mu0=10.0)
    state.y = np.array([1.0, 0.0, 1.0, 0.0])
    state.block_labels = [np.array([1, 0, 1, 0], dtype=np.int8)]
    dope.update_multipliers(state, part, mu_fact=1.05)
    assert np.allclose(state.multipliers[0], 0.0) and state.mu == pytest.approx(10.5)
    state.block_labels = [np.array([1, 1, 1, 0], dtype=np.int8)]
    dope.update_multipliers(state, part, mu_fact=1.0)
    assert np.allclose(state.multipliers[0], [0, 1, 0, 0])
    dope.update_multipliers(state, part, mu_fact=1.0)
    assert np.allclose(state.multipliers[0], [0, 2, 0, 0])
    state.multipliers[0] += 1.0          # in-place edits are what the next step reads
    dope.update_multipliers(state, part, mu_fact=1.0)
    assert np.allclose(state.multipliers[0], [1, 4, 1, 1])


def test_block_solve_error_carries_the_block_id(rng):
    w = dope.SparseWeights(16, [0, 8], [1, 9], [-1.0, 1.0], allow_negative=True)
    model = dope.EnergyModel(rng.normal(size=16), w, lam=1.0)
    part = dope.make_partition(dope.GridShape((4, 4)), (2, 2), 0)
    problems = dope.assemble_block_problems(model, part)
    state = dope.init_state(part, mu0=10.0)
    with pytest.raises(dope.BlockSolveError) as info:
        dope.update_blocks(state, problems, model.lam, dope.AdmmConfig())
    assert info.value.block_id == 0


def test_solve_block_dispatch_and_exhaustive_ties(rng):
    for _ in range(10):
        m = int(rng.integers(1, 12))
        pairs = [(i, j) for i in range(m) for j in range(i + 1, m) if rng.random() < 0.3]
        w = dope.SparseWeights(m, [p[0] for p in pairs], [p[1] for p in pairs], rng.random(len(pairs)))
        lin = rng.normal(size=m)
        a = dope.solve_block(dope.MAXFLOW, lin, w, 1.3)
        b = dope.solve_block(dope.EXHAUSTIVE, lin, w, 1.3)
        assert dope.pairwise_energy(lin, w, 1.3, a) == pytest.approx(dope.pairwise_energy(lin, w, 1.3, b),
                                                                     abs=1e-9)
    labels, e = dope.exhaustive_minimize(np.zeros(5), dope.SparseWeights(5, [], [], []), 1.0)
    assert labels.tolist() == [0] * 5 and e == 0.0   # ties -> lexicographically smallest
    labels, _ = dope.exhaustive_minimize(np.array([0.0, -1.0, 0.0]), dope.SparseWeights(3, [], [], []), 1.0)
    assert labels.tolist() == [0, 1, 0]
    with pytest.raises(NotImplementedError):
        dope.solve_block(dope.ICM, np.zeros(2), dope.SparseWeights(2, [], [], []), 1.0)


def test_evaluate_energy_on_device_matches_numpy(rng):
    model = random_model(rng, (9, 11))
    y = rng.random(model.n)
    w = model.weights
    ref = float(np.dot(model.unary, y)) + model.lam * float(np.dot(w.vals, (y[w.rows] - y[w.cols]) ** 2))
    assert dope.evaluate_energy(model, y) == pytest.approx(ref, rel=1e-13)


def test_run_state_fields_materialise_from_the_device():
    """A lattice run's AdmmState: y / block_labels / multipliers as host arrays on
    first access, consistent with the global-layout helpers."""
    from paper_1704_03116_b200 import workloads as W
    wl = W.mini_disks(128, 32, 4, 2, 8, seed=3, rmax=30.0)
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u.astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0)
    labels, state = dope.run(model, part, dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters))
    yh = state.labels_global()
    for b, lab in zip(part.blocks, state.block_labels):
        assert np.array_equal(lab, yh[b.pixels])
    a = state.multipliers_global()
    for b, m in zip(part.blocks, state.multipliers):
        assert np.array_equal(m, a[b.pixels])
    assert np.array_equal(dope.binarize(state.y), labels)
    # continue the loop through the step API from the run's state
    problems = dope.assemble_block_problems(model, part)
    dope.update_blocks(state, problems, model.lam, dope.AdmmConfig(mu0=1.0, mu_fact=1.0))
    dope.update_global(state, problems, part, model.lam)
    assert state.y.shape == (wl.n,)


def test_repeated_runs_reuse_the_lowering_and_keep_the_graph_cache_bounded():
    """The serving loop of run(): the same weights / partition with new unaries
    reuse the lowering, the device buffers and the captured CUDA graph; 50 runs
    leave the library's graph cache at a constant size; a state that outlives
    the next run keeps its own fields."""
    from paper_1704_03116_b200 import _lib, workloads as W
    wl = W.mini_disks(256, 64, 8, 2, 12, seed=4)
    rows, cols, vals = wl.pair_arrays()
    weights = dope.SparseWeights(wl.n, rows, cols, vals)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    rng = np.random.default_rng(5)
    lb = _lib.lib()
    sizes, first, us = [], None, []
    for i in range(50):
        u = wl.u.astype(np.float64) + rng.integers(-1, 2, wl.n)
        labels, state = dope.run(dope.EnergyModel(u, weights, wl.lam), part, cfg)
        if i == 0:
            first = (u, labels, state, state.y.copy())
        if i in (1, 37):
            us.append((u, labels, [t.energy for t in state.trace]))
        sizes.append(int(lb.dope_graph_cache_entries()))
    assert len(set(sizes[1:])) == 1, sizes
    for u, labels, energies in us:   # a fresh lowering of the same model: identical results
        fresh = dope.run(dope.EnergyModel(u, dope.SparseWeights(wl.n, rows, cols, vals), wl.lam),
                         dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0), cfg)
        assert np.array_equal(fresh[0], labels)
        assert [t.energy for t in fresh[1].trace] == energies
    u0, labels0, state0, y0 = first
    assert np.array_equal(state0.y, y0)                     # survived 49 later runs
    assert np.array_equal(dope.binarize(state0.y), labels0)
    # half-integer unaries leave the integer path: the run falls through to the float kernels
    half = dope.run(dope.EnergyModel(u0 + 0.5, weights, wl.lam), part, cfg)
    ref = dope.run(dope.EnergyModel(u0 + 0.5, dope.SparseWeights(wl.n, rows, cols, vals), wl.lam),
                   dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0), cfg)
    assert np.array_equal(half[0], ref[0])


def test_serving_loop_refilling_one_host_buffer():
    """run() on one host unary buffer refilled in place between calls: from the
    second call the buffer is DMA'd directly (page-locked once), and every
    call sees the new contents -- identical to a fresh lowering each time.
    Switching to another array releases the registration."""
    from paper_1704_03116_b200 import admm as A, workloads as W
    wl = W.mini_disks(256, 64, 8, 2, 10, seed=6)
    rows, cols, vals = wl.pair_arrays()
    weights = dope.SparseWeights(wl.n, rows, cols, vals)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    cfg = dope.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=wl.iters)
    rng = np.random.default_rng(9)
    buf = np.empty(wl.n, dtype=np.float64)
    problems = None
    kept = []      # every returned label array stays alive: the pinned pool must not reuse them
    for i in range(7):
        buf[:] = wl.u + rng.integers(-2, 3, wl.n)
        labels, state = dope.run(dope.EnergyModel(buf, weights, wl.lam), part, cfg)
        fresh = dope.run(dope.EnergyModel(buf.copy(), dope.SparseWeights(wl.n, rows, cols, vals), wl.lam),
                         dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0), cfg)
        assert labels.dtype == np.int8 and np.array_equal(labels, fresh[0])
        assert [t.energy for t in state.trace] == [t.energy for t in fresh[1].trace]
        kept.append((labels, fresh[0].copy()))
        problems = A._problems_for(dope.EnergyModel(buf, weights, wl.lam), part)
    for got, want in kept:
        assert np.array_equal(got, want)
    up = problems._uploader
    assert up.registered_uploads >= 3 and up._registered is not None
    other = buf.copy()
    dope.run(dope.EnergyModel(other, weights, wl.lam), part, cfg)
    assert up._registered is None
