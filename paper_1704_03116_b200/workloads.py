"""Seeded synthetic inputs for the BASELINE.json configs.

The reference measures nothing on public data for this path; these
generators stand in for the paper's images/volumes with the shapes, sizes and
value distributions BASELINE.json names.  One ``numpy.random.default_rng(seed)``
per config, draws in the order documented on each function.

Integer configs (C1, C3, C4, C5) use ``lam = pairwise weight`` and unit
stored weights, so every block capacity is an integer.
Pairs are enumerated direction by direction (horizontal, vertical, then
depth), each i<j in row-major order -- the canonical SparseWeights form of
/root/reference/pkg/src/dope/energy.py:48-53.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# forward stencil offsets (i<j) per connectivity, row-major axes
STENCILS = {
    (2, 4): [(0, 1), (1, 0)],
    (2, 8): [(0, 1), (1, 0), (1, 1), (1, -1)],
    (3, 6): [(0, 0, 1), (0, 1, 0), (1, 0, 0)],
}


@dataclass
class Workload:
    name: str
    dims: tuple                 # row-major grid dims
    block: tuple                # block extent per axis (exact tiling)
    conn: int                   # 4 / 8 (2D) or 6 (3D)
    u: np.ndarray               # unary, flat (int32 for int configs, float64 otherwise)
    weights: list               # per stencil direction: scalar or plane (flat, lower pixel)
    lam: float
    rho: float                  # ADMM penalty mu0 (mu_fact = 1, eps = 0)
    iters: int
    integer: bool
    meta: dict = field(default_factory=dict)

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def n(self) -> int:
        return int(np.prod(self.dims))

    @property
    def kpa(self) -> tuple:
        return tuple(d // b for d, b in zip(self.dims, self.block))

    @property
    def num_blocks(self) -> int:
        return int(np.prod(self.kpa))

    @property
    def offsets(self) -> list:
        return STENCILS[(self.ndim, self.conn)]

    def pair_arrays(self):
        """(rows, cols, vals) in canonical direction-major order (energy.py:48-53)."""
        idx = np.arange(self.n, dtype=np.int64).reshape(self.dims)
        rows, cols, vals = [], [], []
        for off, w in zip(self.offsets, self.weights):
            src = tuple(slice(max(0, -o), d - max(0, o)) for o, d in zip(off, self.dims))
            dst = tuple(slice(max(0, o), d + min(0, o)) for o, d in zip(off, self.dims))
            i = idx[src].ravel()
            j = idx[dst].ravel()
            rows.append(i)
            cols.append(j)
            if np.isscalar(w):
                vals.append(np.full(i.size, float(w)))
            else:
                vals.append(np.asarray(w, dtype=np.float64).ravel()[i])
        return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)

    @property
    def num_pairs(self) -> int:
        e = 0
        for off in self.offsets:
            c = 1
            for o, d in zip(off, self.dims):
                c *= d - abs(o)
            e += c
        return e


def _disk_mask(shape, centres, radii):
    h, w = shape
    mask = np.zeros(shape, dtype=bool)
    for (cy, cx), r in zip(centres, radii):
        y0, y1 = max(0, int(np.floor(cy - r)) - 1), min(h, int(np.ceil(cy + r)) + 2)
        x0, x1 = max(0, int(np.floor(cx - r)) - 1), min(w, int(np.ceil(cx + r)) + 2)
        if y0 >= y1 or x0 >= x1:
            continue
        yy = np.arange(y0, y1, dtype=np.float64)[:, None]
        xx = np.arange(x0, x1, dtype=np.float64)[None, :]
        mask[y0:y1, x0:x1] |= (yy - cy) ** 2 + (xx - cx) ** 2 < r * r
    return mask


def c1(seed: int = 0) -> Workload:
    """256^2 4-conn, centred disk r=80; u = (mask ? -4 : +4) + U{-6..6}; lam*w = 3;
    16 blocks of 64^2; rho = 1; 50 iterations.  Draws: noise."""
    rng = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.arange(256), np.arange(256), indexing="ij")
    mask = (yy - 128) ** 2 + (xx - 128) ** 2 < 80 ** 2
    u = np.where(mask, -4, 4) + rng.integers(-6, 7, (256, 256))
    return Workload("C1", (256, 256), (64, 64), 4, u.astype(np.int32).ravel(), [1, 1],
                    3.0, 1.0, 50, True)


def disks_workload(name, size, ndisks, block, weight, iters, fg=-5, bg=5, noise=8,
                   rmin=20.0, rmax=300.0, seed=0) -> Workload:
    """C3/C5 generator: ndisks disks with centres U[0,size)^2 and radius
    U[rmin,rmax]; u = (mask ? fg : bg) + U{-noise..noise}.
    Draws: centres (ndisks,2), radii (ndisks,), noise (size,size)."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0, size, (ndisks, 2))
    radii = rng.uniform(rmin, rmax, ndisks)
    mask = _disk_mask((size, size), centres, radii)
    u = np.where(mask, fg, bg).astype(np.int32) + \
        rng.integers(-noise, noise + 1, (size, size)).astype(np.int32)
    return Workload(name, (size, size), (block, block), 4, u.ravel(), [1, 1], float(weight),
                    1.0, iters, True, meta={"ndisks": ndisks})


def c3(seed: int = 0) -> Workload:
    """4096^2 4-conn, 64 disks r in [20,300]; u = (mask ? -5 : +5) + U{-8..8};
    weight 2; 4096 blocks of 64^2; rho = 1; 100 iterations."""
    return disks_workload("C3", 4096, 64, 64, 2, 100, seed=seed)


def c5(block: int = 64, seed: int = 0) -> Workload:
    """2048^2, the C3 generator with 32 disks; weight 2; block 16/32/64/128."""
    return disks_workload(f"C5-b{block}", 2048, 32, block, 2, 100, seed=seed)


def c4(seed: int = 0, size: int = 256, block: int = 32, iters: int = 60) -> Workload:
    """256^3 6-conn, union of 8 ellipsoids with centres U[0,256)^3 and
    semi-axes U[16,64]; u = (mask ? -3 : +3) + U{-5..5}; weight 1; 512 blocks of
    32^3; rho = 1; 60 iterations.  Draws: centres (8,3), semi-axes (8,3), noise."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0, size, (8, 3))
    axes = rng.uniform(16 * size / 256, 64 * size / 256, (8, 3))
    mask = np.zeros((size,) * 3, dtype=bool)
    for c, s in zip(centres, axes):
        lo = [max(0, int(np.floor(c[a] - s[a])) - 1) for a in range(3)]
        hi = [min(size, int(np.ceil(c[a] + s[a])) + 2) for a in range(3)]
        if any(l >= h for l, h in zip(lo, hi)):
            continue
        zz = np.arange(lo[0], hi[0], dtype=np.float64)[:, None, None]
        yy = np.arange(lo[1], hi[1], dtype=np.float64)[None, :, None]
        xx = np.arange(lo[2], hi[2], dtype=np.float64)[None, None, :]
        q = ((zz - c[0]) / s[0]) ** 2 + ((yy - c[1]) / s[1]) ** 2 + ((xx - c[2]) / s[2]) ** 2
        mask[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] |= q < 1.0
    u = np.where(mask, -3, 3).astype(np.int32) + rng.integers(-5, 6, mask.shape).astype(np.int32)
    return Workload(f"C4" if size == 256 else f"C4-{size}", (size,) * 3, (block,) * 3, 6,
                    u.ravel(), [1, 1, 1], 1.0, 1.0, iters, True)


def _polygon_mask(shape, ys, xs):
    """Even-odd point-in-polygon over the polygon's bounding box (pixel centres)."""
    h, w = shape
    y0, y1 = max(0, int(np.floor(ys.min()))), min(h, int(np.ceil(ys.max())) + 1)
    x0, x1 = max(0, int(np.floor(xs.min()))), min(w, int(np.ceil(xs.max())) + 1)
    mask = np.zeros(shape, dtype=bool)
    if y0 >= y1 or x0 >= x1:
        return mask
    py = np.arange(y0, y1, dtype=np.float64)[:, None]
    px = np.arange(x0, x1, dtype=np.float64)[None, :]
    inside = np.zeros((y1 - y0, x1 - x0), dtype=bool)
    n = len(ys)
    for k in range(n):
        ya, xa, yb, xb = ys[k], xs[k], ys[(k + 1) % n], xs[(k + 1) % n]
        if ya == yb:
            continue
        cross = (ya > py) != (yb > py)
        xint = (xb - xa) * (py - ya) / (yb - ya) + xa
        inside ^= cross & (px < xint)
    mask[y0:y1, x0:x1] = inside
    return mask


def c2(seed: int = 0, size: int = 1024, block: int = 64, iters: int = 100) -> Workload:
    """1024^2 8-conn contrast-sensitive Potts (float): background colour U[0,1]^3;
    12 star polygons (3..8 vertices, radius U[0.04,0.16]*size around a centre
    U[0,size)^2, colour U[0,1]^3); + N(0, 0.08^2) noise, not clipped; fixed
    Gaussian colour models (fg mean = mean polygon colour, bg mean = background
    colour, isotropic sigma_c = 0.25): u = loglik_bg - loglik_fg
    (energy.py:315-316 convention); w = exp(-|x_i-x_j|^2 / (2*0.1^2)) / dist;
    lam = 2.0; blocks of 64^2; rho = 0.5; 100 iterations.  u and w rounded to
    float32.  Draws: background, then per polygon (nv,
    centre, radii, angles, colour), then the noise."""
    rng = np.random.default_rng(seed)
    bg = rng.uniform(0, 1, 3)
    img = np.empty((size, size, 3))
    img[:] = bg
    cols = []
    for _ in range(12):
        nv = int(rng.integers(3, 9))
        cy, cx = rng.uniform(0, size, 2)
        rad = rng.uniform(0.04, 0.16, nv) * size
        ang = np.sort(rng.uniform(0, 2 * np.pi, nv))
        col = rng.uniform(0, 1, 3)
        mask = _polygon_mask((size, size), cy + rad * np.sin(ang), cx + rad * np.cos(ang))
        img[mask] = col
        cols.append(col)
    img += rng.normal(0.0, 0.08, img.shape)
    fg = np.mean(cols, axis=0)
    sc = 0.25
    u = (((img - fg) ** 2).sum(-1) - ((img - bg) ** 2).sum(-1)) / (2 * sc * sc)
    u = u.astype(np.float32).astype(np.float64).ravel()
    planes = []
    for off in STENCILS[(2, 8)]:
        dy, dx = off
        dist = np.sqrt(dy * dy + dx * dx)
        wpl = np.zeros((size, size))
        ys = slice(0, size - dy)
        xs = slice(max(0, -dx), size - max(0, dx))
        yd = slice(dy, size)
        xd = slice(max(0, dx), size + min(0, dx))
        d2 = ((img[ys, xs] - img[yd, xd]) ** 2).sum(-1)
        wpl[ys, xs] = np.exp(-d2 / (2 * 0.1 * 0.1)) / dist
        planes.append(wpl.astype(np.float32).astype(np.float64).ravel())
    return Workload("C2" if size == 1024 else f"C2-{size}", (size, size), (block, block), 8, u,
                    planes, 2.0, 0.5, iters, False)


def mini_disks(size=256, block=64, ndisks=8, weight=2, iters=20, seed=0, rmax=80.0) -> Workload:
    """Small C3-like case for parity tests (oracle finishes in seconds)."""
    return disks_workload(f"mini{size}-b{block}", size, ndisks, block, weight, iters,
                          rmin=8.0, rmax=rmax, seed=seed)


def by_name(name: str, seed: int = 0) -> Workload:
    name = name.upper()
    if name == "C1":
        return c1(seed)
    if name == "C3":
        return c3(seed)
    if name == "C4":
        return c4(seed)
    if name == "C2":
        return c2(seed)
    if name == "C2-OV25":
        # general path: C2's image on 32^2 blocks grown by
        # 25 % (q in {1, 2, 4}), the reference's default growing mu (mu0 100,
        # mu_fact 1.05), eps = 0 so every run does its 50 iterations
        wl = c2(seed, size=1024, block=32, iters=50)
        wl.name = "C2-ov25"
        wl.meta = dict(wl.meta or {}, overlap=25, mu0=100.0, mu_fact=1.05)
        return wl
    if name.startswith("C5"):
        b = int(name.split("-B")[-1]) if "-B" in name else 64
        return c5(b, seed)
    raise KeyError(name)
