"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src and routes its
max-flow seam to the reference's own compiled core (oracle/_ref, built from
_core.pyx by oracle/build_oracle.py) exactly as the reference's benchmark
swaps backends (pkg/benchmarks/bench_backends.py:42-44).  Outputs are small
.npz files committed to the repo; nothing at test time reads /root/reference.

Fixtures
  bk_graphs.npz   random single graphs (test_backends.py:12-25 and
                  test_maxflow.py:65-76 styles, plus integer lattices) with the
                  reference's labels and flow values.
  run_<case>.npz  full admm.run traces: per-iteration mu, energy, residual_sq,
                  max_block_residual, clamped, block labels (packed bits), plus
                  the final state.y, labels, multipliers, converged, iterations,
                  best_iteration.  Config mapping of SURVEY.md §8(a):
                  AdmmConfig(mu0=rho, mu_fact=1, eps=0, max_iters=N).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, "/root/reference/pkg/src")

import dope  # noqa: E402  (the reference)
import dope.admm as ref_admm  # noqa: E402
import dope.maxflow as ref_maxflow  # noqa: E402
from dope.energy import EnergyModel, SparseWeights  # noqa: E402
from dope.grid import GridShape  # noqa: E402
from dope.partition import make_partition  # noqa: E402

import build_oracle  # noqa: E402
from paper_1704_03116_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent


def ref_core():
    build_oracle.build_reference_core()
    import oracle as orc  # noqa
    core = orc.reference_core()
    assert core is not None and core.BACKEND == "compiled"
    return core


def gen_bk(core):
    rng = np.random.default_rng(20261019)
    graphs = []
    # test_backends.py:12-25 style (float caps, directed asymmetric)
    for _ in range(150):
        m = int(rng.integers(1, 40))
        pairs = [(i, j) for i in range(m) for j in range(i + 1, m) if rng.random() < 0.25]
        pi = np.array([p[0] for p in pairs], dtype=np.int32)
        pj = np.array([p[1] for p in pairs], dtype=np.int32)
        cij = rng.random(pi.size) * 3
        cji = rng.random(pi.size) * 3
        tcap = rng.uniform(-4, 4, m)
        if rng.random() < 0.3:
            tcap = np.round(tcap)
        graphs.append((tcap, pi, pj, cij, cji))
    # integer instances with many exact ties (tie-break pinning)
    for _ in range(150):
        m = int(rng.integers(1, 64))
        pairs = [(i, j) for i in range(m) for j in range(i + 1, m) if rng.random() < 0.15]
        pi = np.array([p[0] for p in pairs], dtype=np.int32)
        pj = np.array([p[1] for p in pairs], dtype=np.int32)
        c = rng.integers(0, 4, pi.size).astype(np.float64)
        asym = rng.random() < 0.3
        cji = rng.integers(0, 4, pi.size).astype(np.float64) if asym else c.copy()
        tcap = rng.integers(-3, 4, m).astype(np.float64)
        graphs.append((tcap, pi, pj, c, cji))
    # small integer lattices (the block problems' shape)
    for _ in range(40):
        h, w = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        idx = np.arange(h * w).reshape(h, w)
        pi = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()]).astype(np.int32)
        pj = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()]).astype(np.int32)
        c = np.full(pi.size, float(rng.integers(1, 5)))
        tcap = rng.integers(-8, 9, h * w).astype(np.float64)
        graphs.append((tcap, pi, pj, c, c.copy()))
    # empty graph and isolated nodes
    graphs.append((np.zeros(0), np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0), np.zeros(0)))
    graphs.append((np.array([0.0, -1.0, 2.0, 0.0]), np.zeros(0, np.int32), np.zeros(0, np.int32),
                   np.zeros(0), np.zeros(0)))
    labels, flows = [], []
    for g in graphs:
        lab, fl = core.bk_maxflow(g[0].copy(), *g[1:])
        labels.append(np.asarray(lab, dtype=np.uint8))
        flows.append(fl)
    m_off = np.cumsum([0] + [g[0].size for g in graphs])
    p_off = np.cumsum([0] + [g[1].size for g in graphs])
    np.savez_compressed(
        OUT / "bk_graphs.npz",
        m_off=m_off, p_off=p_off,
        tcap=np.concatenate([g[0] for g in graphs]),
        pi=np.concatenate([g[1] for g in graphs]).astype(np.int32),
        pj=np.concatenate([g[2] for g in graphs]).astype(np.int32),
        cij=np.concatenate([g[3] for g in graphs]),
        cji=np.concatenate([g[4] for g in graphs]),
        labels=np.concatenate(labels), flows=np.array(flows))
    print("bk_graphs:", len(graphs))


def ref_run(wl: W.Workload, iters: int | None = None):
    rows, cols, vals = wl.pair_arrays()
    shape = GridShape(wl.dims)
    model = EnergyModel(wl.u.astype(np.float64), SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = make_partition(shape, wl.kpa, 0)
    cfg = ref_admm.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0,
                              max_iters=iters if iters else wl.iters)
    hist = []
    orig = ref_admm.update_blocks

    def recording(state, problems, lam, config):
        out = orig(state, problems, lam, config)
        g = np.zeros(wl.n, dtype=np.uint8)
        for b, lab in zip(part.blocks, state.block_labels):
            g[b.pixels] = lab
        hist.append(g)
        return out

    ref_admm.update_blocks = recording
    try:
        labels, state = ref_admm.run(model, part, cfg)
    finally:
        ref_admm.update_blocks = orig
    a = np.zeros(wl.n)
    for b, m in zip(part.blocks, state.multipliers):
        a[b.pixels] = m
    tr = state.trace
    return dict(
        mu=np.array([t.mu for t in tr]), energy=np.array([t.energy for t in tr]),
        residual_sq=np.array([t.residual_sq for t in tr]),
        max_block_residual=np.array([t.max_block_residual for t in tr]),
        clamped=np.array([t.clamped for t in tr]),
        yhat_bits=np.packbits(np.array(hist, dtype=np.uint8), axis=1),
        y=state.y, labels=np.asarray(labels, dtype=np.int8), a=a,
        converged=state.converged, iterations=state.iteration,
        best_iteration=state.best_iteration)


def save_run(case: str, wl: W.Workload, iters: int | None = None, store_u: bool = True):
    r = ref_run(wl, iters)
    meta = dict(dims=np.array(wl.dims), block=np.array(wl.block), conn=wl.conn, lam=wl.lam,
                rho=wl.rho, max_iters=iters if iters else wl.iters, name=wl.name)
    if store_u:
        meta["u"] = wl.u
    if not wl.integer:
        meta["wplanes"] = np.stack([np.asarray(w, dtype=np.float64) for w in wl.weights])
    np.savez_compressed(OUT / f"run_{case}.npz", **r, **meta)
    print(f"run_{case}: iters={r['iterations']} converged={r['converged']} "
          f"best={r['best_iteration']} E_last={r['energy'][-1]}")


def ref_run_general(wl: W.Workload, overlap: int, mu0, mu_fact: float, eps, iters: int):
    """admm.run on an (optionally overlapping) partition with an arbitrary mu
    schedule; per-copy block labels / multipliers in block order."""
    rows, cols, vals = wl.pair_arrays()
    shape = GridShape(wl.dims)
    model = EnergyModel(wl.u.astype(np.float64), SparseWeights(wl.n, rows, cols, vals), wl.lam)
    part = make_partition(shape, wl.kpa, overlap)
    cfg = ref_admm.AdmmConfig(mu0=mu0, mu_fact=mu_fact, eps=eps, max_iters=iters)
    hist = []
    orig = ref_admm.update_blocks

    def recording(state, problems, lam, config):
        out = orig(state, problems, lam, config)
        hist.append(np.concatenate([np.asarray(l, dtype=np.uint8) for l in state.block_labels]))
        return out

    ref_admm.update_blocks = recording
    try:
        labels, state = ref_admm.run(model, part, cfg)
    finally:
        ref_admm.update_blocks = orig
    tr = state.trace
    return dict(
        mu=np.array([t.mu for t in tr]), energy=np.array([t.energy for t in tr]),
        residual_sq=np.array([t.residual_sq for t in tr]),
        max_block_residual=np.array([t.max_block_residual for t in tr]),
        clamped=np.array([t.clamped for t in tr]),
        yhat_bits=np.packbits(np.array(hist, dtype=np.uint8), axis=1),
        y=state.y, labels=np.asarray(labels, dtype=np.int8),
        a_copies=np.concatenate([np.asarray(m, dtype=np.float64) for m in state.multipliers]),
        converged=state.converged, iterations=state.iteration,
        best_iteration=state.best_iteration, counts=part.counts,
        eps=cfg.resolved_eps(part), mu0=cfg.resolved_mu0(shape.ndim))


def save_general(case: str, wl: W.Workload, overlap: int, mu0, mu_fact: float, eps, iters: int):
    r = ref_run_general(wl, overlap, mu0, mu_fact, eps, iters)
    meta = dict(dims=np.array(wl.dims), block=np.array(wl.block), conn=wl.conn, lam=wl.lam,
                overlap=overlap, mu_fact=mu_fact, max_iters=iters, name=wl.name, u=wl.u,
                wplanes=np.stack([np.asarray(w, dtype=np.float64) for w in wl.weights]))
    np.savez_compressed(OUT / f"gen_{case}.npz", **r, **meta)
    print(f"gen_{case}: iters={r['iterations']} converged={r['converged']} "
          f"best={r['best_iteration']} E_last={r['energy'][-1]} qmax={int(r['counts'].max())}")


def main_general():
    """General path: overlapping partitions (q in {1,2,4})
    and the reference's default mu schedule (mu_fact = 1.05, eps from the
    block size)."""
    # contrast-weighted 8-conn image, 4x4 blocks grown by 25 %, default config
    save_general("c2ov25", W.c2(size=64, block=16, iters=50), 25, None, 1.05, None, 50)
    save_general("c2ov25_long", W.c2(size=64, block=16, iters=25), 25, None, 1.05, 0.0, 25)
    # integer 4-conn disks, 4x4 blocks grown by 10 %, fixed mu (lam*w/mu = 2)
    ov = W.mini_disks(128, 32, 6, 2, 20, seed=8, rmax=40.0)
    save_general("int_ov10", ov, 10, 1.0, 1.0, 0.0, 20)
    # non-overlapping tiling with the default growing mu and eps (converges)
    save_general("mufact", W.mini_disks(128, 32, 6, 2, 50, seed=9, rmax=40.0), 0, None, 1.05, None, 50)
    save_general("mufact_long", W.mini_disks(128, 32, 6, 2, 20, seed=9, rmax=40.0), 0, 4.0, 1.05, 0.0, 20)


def main_inputs():
    """Model construction: the reference's weight,
    sigma, colour-model and unary builders on small synthetic images."""
    from dope.energy import build_potts_weights, compute_unaries, estimate_sigma, fit_color_model
    from dope.grid import GridImage
    rng = np.random.default_rng(31)
    h, w = 48, 64
    yy, xx = np.meshgrid(np.arange(h), np.arange(w), indexing="ij")
    blob = ((yy - 20.0) ** 2 / 120.0 + (xx - 30.0) ** 2 / 300.0) < 1.0
    rgb = np.where(blob[..., None], [0.8, 0.3, 0.2], [0.2, 0.5, 0.7]) + rng.normal(0, 0.07, (h, w, 3))
    seeds = np.zeros((h, w), dtype=np.int8)
    seeds[18:22, 24:36] = 2          # foreground strokes
    seeds[2:4, 2:60] = 1             # background strokes
    seeds[44:46, 10:50] = 1
    img = GridImage(GridShape((h, w)), np.clip(rgb, 0, 1).reshape(-1, 3), seeds.ravel())
    out = dict(data=img.data, seeds=img.seeds, dims=np.array((h, w)))
    for k in (3, 5):
        s = estimate_sigma(img, k)
        wts = build_potts_weights(img, k, s, contrast=True)
        out[f"sigma{k}"] = s
        out[f"rows{k}"], out[f"cols{k}"], out[f"vals{k}"] = wts.rows, wts.cols, wts.vals
    cm = fit_color_model(img, rng=np.random.default_rng(0))
    out.update(fg_c=cm.fg_centroids, bg_c=cm.bg_centroids, fg_w=cm.fg_weights, bg_w=cm.bg_weights,
               bw=cm.bandwidth, u=compute_unaries(img, cm))
    np.savez_compressed(OUT / "inputs_2d.npz", **out)
    vol = np.clip(0.5 + 0.3 * np.sin(np.arange(12 * 10 * 8) * 0.37) + rng.normal(0, 0.05, 960), 0, 1)
    img3 = GridImage(GridShape((12, 10, 8)), vol)
    out3 = dict(data=img3.data, dims=np.array((12, 10, 8)))
    for k in (3, 5):
        s = estimate_sigma(img3, k)
        wts = build_potts_weights(img3, k, s, contrast=True)
        out3[f"sigma{k}"] = s
        out3[f"rows{k}"], out3[f"cols{k}"], out3[f"vals{k}"] = wts.rows, wts.cols, wts.vals
    np.savez_compressed(OUT / "inputs_3d.npz", **out3)
    print("inputs:", {k: out[f"vals{k}"].size for k in (3, 5)}, {k: out3[f"vals{k}"].size for k in (3, 5)})


def ref_run_model(model, part, cfg):
    """admm.run of an arbitrary reference model / partition / config, with every
    iteration's per-copy block labels (block order)."""
    hist = []
    orig = ref_admm.update_blocks

    def recording(state, problems, lam, config):
        out = orig(state, problems, lam, config)
        hist.append(np.concatenate([np.asarray(l, dtype=np.uint8) for l in state.block_labels]))
        return out

    ref_admm.update_blocks = recording
    try:
        labels, state = ref_admm.run(model, part, cfg)
    finally:
        ref_admm.update_blocks = orig
    tr = state.trace
    return dict(
        mu=np.array([t.mu for t in tr]), energy=np.array([t.energy for t in tr]),
        residual_sq=np.array([t.residual_sq for t in tr]),
        max_block_residual=np.array([t.max_block_residual for t in tr]),
        clamped=np.array([t.clamped for t in tr]),
        yhat_bits=np.packbits(np.array(hist, dtype=np.uint8), axis=1),
        y=state.y, labels=np.asarray(labels, dtype=np.int8),
        a_copies=np.concatenate([np.asarray(m, dtype=np.float64) for m in state.multipliers]),
        converged=state.converged, iterations=state.iteration,
        best_iteration=state.best_iteration, counts=part.counts,
        eps=cfg.resolved_eps(part), mu0=cfg.resolved_mu0(part.shape.ndim))


def save_graph(case, model, shape, kpa, overlap, cfg, integer):
    part = make_partition(shape, kpa, overlap)
    r = ref_run_model(model, part, cfg)
    w = model.weights
    meta = dict(dims=np.array(shape.dims), kpa=np.array(kpa), overlap=overlap,
                u=model.unary, rows=w.rows, cols=w.cols, vals=w.vals, lam=model.lam,
                cfg_mu0=np.nan if cfg.mu0 is None else cfg.mu0, cfg_mu_fact=cfg.mu_fact,
                cfg_eps=np.nan if cfg.eps is None else cfg.eps, max_iters=cfg.max_iters,
                integer=integer)
    np.savez_compressed(OUT / f"graph_{case}.npz", **r, **meta)
    print(f"graph_{case}: iters={r['iterations']} converged={r['converged']} "
          f"best={r['best_iteration']} E_last={r['energy'][-1]} qmax={int(r['counts'].max())}")


def main_graph():
    """The general graph path: models / partitions the lattice kernels do not
    take -- 3D overlap (q up to 8), the 3D default config, kernel-5 windows."""
    from dope.energy import build_potts_weights
    from dope.grid import GridImage
    # 3D 6-connected integer model, 2x2x2 blocks grown by 25 %, fixed integer mu
    wl = W.c4(seed=12, size=24, block=12, iters=15)
    rows, cols, vals = wl.pair_arrays()
    m3 = EnergyModel(wl.u.astype(np.float64), SparseWeights(wl.n, rows, cols, vals), 2.0)
    save_graph("int3d_ov25", m3, GridShape(wl.dims), (2, 2, 2), 25,
               ref_admm.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=15), True)
    # the same volume, 10 % overlap, q in {1, 2, 4, 8}
    save_graph("int3d_ov10", m3, GridShape(wl.dims), (3, 2, 2), 10,
               ref_admm.AdmmConfig(mu0=2.0, mu_fact=1.0, eps=0.0, max_iters=12), True)
    # the reference's DEFAULT config on a 3D integer model (mu0 500, mu_fact 1.05, eps)
    save_graph("int3d_default", m3, GridShape(wl.dims), (2, 2, 2), 0,
               ref_admm.AdmmConfig(max_iters=20), False)
    # 2D kernel-5 contrast window (non-lattice pair set), 2x3 blocks, 10 % overlap, default
    rng = np.random.default_rng(41)
    h, wd = 40, 36
    yy, xx = np.meshgrid(np.arange(h), np.arange(wd), indexing="ij")
    fg = ((yy - 18.0) ** 2 + (xx - 20.0) ** 2) < 110.0
    img = GridImage(GridShape((h, wd)), np.clip(np.where(fg, 0.75, 0.3) + rng.normal(0, 0.08, (h, wd)),
                                                0, 1).ravel())
    wts = build_potts_weights(img, 5, sigma=0.2, contrast=True)
    mk = EnergyModel((0.5 - img.data[:, 0]) * 8.0, wts, 1.5)
    save_graph("k5_ov10", mk, GridShape((h, wd)), (2, 3), 10, ref_admm.AdmmConfig(max_iters=30), False)
    save_graph("k5_sched", mk, GridShape((h, wd)), (3, 3), 25,
               ref_admm.AdmmConfig(mu0=2.0, mu_fact=1.05, eps=0.0, max_iters=25), False)
    # 3D kernel-3 window (18-connected) with unit weights and integer unaries, 25 % overlap
    v3 = GridImage(GridShape((10, 12, 14)), np.zeros(10 * 12 * 14))
    w3 = build_potts_weights(v3, 3, sigma=1.0, contrast=False)
    u3 = rng.integers(-4, 5, v3.shape.n).astype(np.float64)
    save_graph("int3d_k3_ov25", EnergyModel(u3, w3, 1.0), v3.shape, (2, 2, 2), 25,
               ref_admm.AdmmConfig(mu0=1.0, mu_fact=1.0, eps=0.0, max_iters=10), True)


class _RaggedWL(W.Workload):
    @property
    def kpa(self):
        return self.meta["kpa"]


def main():
    core = ref_core()
    ref_maxflow.bk_maxflow = core.bk_maxflow     # the reference's own seam swap
    if "--only-float" in sys.argv:
        save_run("c2mini", W.c2(size=128, block=32, iters=30))
        return
    if "--only-general" in sys.argv:
        main_general()
        return
    if "--only-inputs" in sys.argv:
        main_inputs()
        return
    if "--only-graph" in sys.argv:
        main_graph()
        return
    gen_bk(core)
    save_run("c1", W.c1())
    save_run("mini256", W.mini_disks(256, 64, 8, 2, 25, seed=1))
    save_run("mini128_b16", W.mini_disks(128, 16, 6, 2, 20, seed=2, rmax=40.0))
    save_run("mini256_b128", W.mini_disks(256, 128, 6, 2, 15, seed=3))
    save_run("mini3d", W.c4(seed=4, size=64, block=32, iters=12))
    rng = np.random.default_rng(7)
    rag = _RaggedWL("ragged70x53", (70, 53), (0, 0), 4,
                    rng.integers(-6, 7, (70, 53)).astype(np.int32).ravel(), [1, 1], 2.0, 1.0,
                    12, True, meta={"kpa": (3, 4)})
    r = ref_run(rag)
    np.savez_compressed(OUT / "run_ragged.npz", **r, dims=np.array(rag.dims),
                        kpa=np.array((3, 4)), conn=4, lam=2.0, rho=1.0, max_iters=12,
                        name=rag.name, u=rag.u)
    print("run_ragged:", r["iterations"], r["energy"][-1])
    # early convergence (stop rule admm.py:247-249): one block converges at it 1
    one = W.mini_disks(64, 64, 2, 1, 10, seed=5, rmax=20.0)
    save_run("single_block", one)
    # float config C2 (8-conn contrast weights, rho = 0.5) at 128^2 with 16 blocks
    if "--only-float" in sys.argv or True:
        save_run("c2mini", W.c2(size=128, block=32, iters=30))
    # rho = 2 with lam*w = 2: lam/mu = 1 stays integral
    r2 = W.mini_disks(128, 32, 4, 2, 15, seed=6, rmax=40.0)
    r2.rho = 2.0
    save_run("rho2", r2)
    main_general()
    main_inputs()
    main_graph()


if __name__ == "__main__":
    main()
