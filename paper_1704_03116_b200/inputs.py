"""Model construction on the GPU.

Same names and semantics as the reference's energy.py / grid.py builders:

* ``build_potts_weights(image, kernel, sigma, contrast)`` (energy.py:124-162):
  pairs of the half window (grid.py:80-116) enumerated per offset over the
  clipped source region, contrast weights exp(-|x_i - x_j|^2 / (2 sigma^2)),
  computed by ``dope_in_potts_weights``;
* ``estimate_sigma(image, kernel)`` (energy.py:165-184): RMS neighbour
  difference, reduced on the GPU;
* ``fit_color_model`` / ``kmeans`` (energy.py:220-287): k-means on the seed
  pixels only (a few hundred points), on the host with the reference's
  algorithm and random draws;
* ``compute_unaries(image, model)`` (energy.py:298-323): per-pixel mixture
  log-likelihood ratio with seed pinning, ``dope_in_unaries``.

Results match the reference to floating-point rounding (exp / log); there is
no CPU fallback for the per-pixel work.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from . import _lib
from .energy import SparseWeights
from .grid import GridShape

SUPPORTED_KERNELS = (3, 5, 7, 9)
SEED_NONE, SEED_BG, SEED_FG = 0, 1, 2
N_COLOR_CLUSTERS = 5


@dataclass
class GridImage:
    """Per-pixel feature vectors (n, channels) in [0, 1] plus optional seeds."""
    shape: GridShape
    data: np.ndarray
    seeds: np.ndarray | None = field(default=None)

    def __post_init__(self):
        self.data = np.asarray(self.data, dtype=np.float64)
        if self.data.ndim == 1:
            self.data = self.data[:, None]
        if self.data.shape[0] != self.shape.n:
            raise ValueError(f"data has {self.data.shape[0]} rows, expected n={self.shape.n}")
        if self.seeds is not None:
            self.seeds = np.asarray(self.seeds, dtype=np.int8)
            if self.seeds.shape != (self.shape.n,):
                raise ValueError(f"seed vector has shape {self.seeds.shape}, expected ({self.shape.n},)")
            if not np.isin(self.seeds, (SEED_NONE, SEED_BG, SEED_FG)).all():
                raise ValueError("seed values must be 0 (none), 1 (background) or 2 (foreground)")

    @property
    def channels(self) -> int:
        return int(self.data.shape[1])


@lru_cache(maxsize=None)
def kernel_offsets(ndim: int, kernel: int) -> tuple:
    """2D: the full square window of side `kernel`; 3D: the discrete ball of
    radius kernel/2 (grid.py:80-110); centre excluded."""
    if kernel not in SUPPORTED_KERNELS:
        raise ValueError(f"unsupported kernel size {kernel}, expected one of {SUPPORTED_KERNELS}")
    h = (kernel - 1) // 2
    r = range(-h, h + 1)
    if ndim == 2:
        return tuple((a, b) for a in r for b in r if (a, b) != (0, 0))
    if ndim == 3:
        lim = (kernel / 2.0) ** 2
        return tuple((a, b, c) for a in r for b in r for c in r
                     if (a, b, c) != (0, 0, 0) and a * a + b * b + c * c <= lim)
    raise ValueError(f"unsupported dimensionality {ndim}")


def half_kernel_offsets(ndim: int, kernel: int) -> tuple:
    return tuple(o for o in kernel_offsets(ndim, kernel) if o > (0,) * ndim)


def _device():
    import torch
    return torch.device("cuda", torch.cuda.current_device())


def _stream(dev):
    import torch
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _check(rc, what):
    if rc == _lib.DOPE_E_CUDA:
        raise _lib.DopeError(f"{what} failed: {_lib.lib().dope_in_last_error().decode()}")
    _lib.check(rc, what)


def _window(shape: GridShape, kernel: int):
    offs = np.ascontiguousarray(half_kernel_offsets(shape.ndim, kernel), dtype=np.int32).ravel()
    dims = (C.c_int64 * 3)(*[int(d) for d in shape.dims])
    return offs, dims, len(offs) // shape.ndim


def build_potts_weights(image: GridImage, kernel: int, sigma: float, contrast: bool = True) -> SparseWeights:
    import torch
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    shape = image.shape
    offs, dims, noff = _window(shape, kernel)
    lb = _lib.lib()
    po = offs.ctypes.data_as(C.POINTER(C.c_int32))
    total = int(lb.dope_in_pair_count(shape.ndim, dims, noff, po))
    if total <= 0:
        return SparseWeights(shape.n, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    dev = _device()
    data = torch.as_tensor(np.ascontiguousarray(image.data), device=dev)
    rows = torch.empty(total, dtype=torch.int64, device=dev)
    cols = torch.empty(total, dtype=torch.int64, device=dev)
    vals = torch.empty(total, dtype=torch.float64, device=dev)
    _check(lb.dope_in_potts_weights(shape.ndim, dims, image.channels, data.data_ptr(), noff, po, float(sigma),
                                    int(bool(contrast)), rows.data_ptr(), cols.data_ptr(), vals.data_ptr(),
                                    _stream(dev)), "dope_in_potts_weights")
    return SparseWeights(shape.n, rows.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy())


def estimate_sigma(image: GridImage, kernel: int) -> float:
    import torch
    shape = image.shape
    offs, dims, noff = _window(shape, kernel)
    lb = _lib.lib()
    po = offs.ctypes.data_as(C.POINTER(C.c_int32))
    count = int(lb.dope_in_pair_count(shape.ndim, dims, noff, po))
    if count <= 0:
        return 1.0
    dev = _device()
    data = torch.as_tensor(np.ascontiguousarray(image.data), device=dev)
    part = torch.zeros(int(lb.dope_in_partials(count)), dtype=torch.float64, device=dev)
    _check(lb.dope_in_sq_diff(shape.ndim, dims, image.channels, data.data_ptr(), noff, po, part.data_ptr(),
                              _stream(dev)), "dope_in_sq_diff")
    ms = float(part.sum().item()) / count
    return float(np.sqrt(ms)) if ms > 1e-12 else 1.0


@dataclass
class ColorModel:
    fg_centroids: np.ndarray
    bg_centroids: np.ndarray
    fg_weights: np.ndarray
    bg_weights: np.ndarray
    bandwidth: float


def _lloyd(points: np.ndarray, k: int, rng: np.random.Generator, max_iters: int, tol: float):
    """One Lloyd run (energy.py:220-250): random distinct initial centres,
    argmin ties to the lowest index, empty clusters take the farthest point."""
    cent = points[rng.choice(points.shape[0], size=k, replace=False)].copy()
    for _ in range(max_iters):
        d2 = ((points[:, None, :] - cent[None, :, :]) ** 2).sum(axis=2)
        assign = np.argmin(d2, axis=1)
        new = cent.copy()
        for c in range(k):
            sel = assign == c
            if sel.any():
                new[c] = points[sel].mean(axis=0)
        far_d = d2[np.arange(points.shape[0]), assign]
        for c in range(k):
            if not (assign == c).any():
                f = int(np.argmax(far_d))
                new[c] = points[f]
                far_d[f] = -np.inf
        move = float(np.max(np.abs(new - cent)))
        cent = new
        if move <= tol:
            break
    d2 = ((points[:, None, :] - cent[None, :, :]) ** 2).sum(axis=2)
    assign = np.argmin(d2, axis=1)
    return cent, assign, float(d2[np.arange(points.shape[0]), assign].sum())


def kmeans(points, k: int = N_COLOR_CLUSTERS, restarts: int = 10, max_iters: int = 100, tol: float = 1e-6,
           rng: np.random.Generator | None = None):
    rng = np.random.default_rng(0) if rng is None else rng
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    if pts.shape[0] < k:
        raise ValueError(f"need at least {k} points, got {pts.shape[0]}")
    best = None
    for _ in range(restarts):
        cand = _lloyd(pts, k, rng, max_iters, tol)
        if best is None or cand[2] < best[2]:
            best = cand
    return best


def fit_color_model(image: GridImage, rng: np.random.Generator | None = None) -> ColorModel:
    if image.seeds is None:
        raise ValueError("image has no seed mask")
    rng = np.random.default_rng(0) if rng is None else rng
    fg = image.data[image.seeds == SEED_FG]
    bg = image.data[image.seeds == SEED_BG]
    if fg.shape[0] < N_COLOR_CLUSTERS or bg.shape[0] < N_COLOR_CLUSTERS:
        raise ValueError(f"need at least {N_COLOR_CLUSTERS} seeds per class, got fg={fg.shape[0]} bg={bg.shape[0]}")
    fg_c, fg_a, _ = kmeans(fg, rng=rng)
    bg_c, bg_a, _ = kmeans(bg, rng=rng)
    fg_w = np.bincount(fg_a, minlength=N_COLOR_CLUSTERS) / fg.shape[0]
    bg_w = np.bincount(bg_a, minlength=N_COLOR_CLUSTERS) / bg.shape[0]
    d_fg = np.sqrt(((fg[:, None, :] - fg_c[None]) ** 2).sum(axis=2)).min(axis=1)
    d_bg = np.sqrt(((bg[:, None, :] - bg_c[None]) ** 2).sum(axis=2)).min(axis=1)
    bw = max(float(np.concatenate([d_fg, d_bg]).mean()), 1e-6)
    return ColorModel(fg_c, bg_c, fg_w, bg_w, bw)


def compute_unaries(image: GridImage, model: ColorModel) -> np.ndarray:
    import torch
    dev = _device()
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    data = t(image.data)
    n = image.shape.n
    u = torch.empty(n, dtype=torch.float64, device=dev)
    lb = _lib.lib()
    part = torch.zeros(int(lb.dope_in_partials(n)), dtype=torch.float64, device=dev)
    seeds = torch.as_tensor(image.seeds, device=dev) if image.seeds is not None else None
    fgc, bgc, fgw, bgw = t(model.fg_centroids), t(model.bg_centroids), t(model.fg_weights), t(model.bg_weights)
    _check(lb.dope_in_unaries(n, image.channels, data.data_ptr(), seeds.data_ptr() if seeds is not None else None,
                              fgc.data_ptr(), bgc.data_ptr(), fgw.data_ptr(), bgw.data_ptr(),
                              int(model.fg_centroids.shape[0]), float(model.bandwidth), u.data_ptr(),
                              part.data_ptr(), _stream(dev)), "dope_in_unaries")
    return u.cpu().numpy()
