"""Grid geometry: the row-major pixel numbering every device array uses.

Mirrors the reference's GridShape (grid.py:21-77): 2D (H, W) or 3D (D, H, W)
grids, pixel g = sum_a coord_a * stride_a with the last axis fastest, so each
device vector compares elementwise with the reference's global vectors.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import reduce


def _row_major_strides(dims) -> tuple:
    out = []
    step = 1
    for d in reversed(dims):
        out.append(step)
        step *= d
    return tuple(reversed(out))


@dataclass(frozen=True)
class GridShape:
    """Extents of a 2D / 3D pixel grid (reference grid.py:21-52)."""

    dims: tuple

    def __post_init__(self):
        ext = tuple(int(d) for d in self.dims)
        if not 2 <= len(ext) <= 3:
            raise ValueError(f"grid must be 2D or 3D, got {len(ext)} axes")
        if min(ext) < 1:
            raise ValueError(f"all grid dimensions must be positive, got {ext}")
        object.__setattr__(self, "dims", ext)

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def n(self) -> int:
        return reduce(lambda a, b: a * b, self.dims, 1)

    @property
    def strides(self) -> tuple:
        return _row_major_strides(self.dims)


def index_of(shape: GridShape, coords) -> int:
    """Linear index of a coordinate tuple (grid.py:55-66)."""
    c = tuple(int(v) for v in coords)
    if len(c) != shape.ndim:
        raise ValueError(f"expected {shape.ndim} coordinates, got {len(c)}")
    if any(not 0 <= v < d for v, d in zip(c, shape.dims)):
        raise ValueError(f"coordinate {c} outside grid {shape.dims}")
    return sum(v * s for v, s in zip(c, shape.strides))


def coords_of(shape: GridShape, index: int) -> tuple:
    """Coordinate tuple of a linear index (grid.py:69-77)."""
    g = int(index)
    if not 0 <= g < shape.n:
        raise ValueError(f"index {g} outside grid of {shape.n} pixels")
    coords = []
    for d in reversed(shape.dims):
        g, r = divmod(g, d)
        coords.append(r)
    return tuple(reversed(coords))
