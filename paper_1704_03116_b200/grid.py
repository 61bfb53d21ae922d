"""Grid shapes and row-major indexing (mirror of reference grid.py:21-77).

Only the parts the hot path needs: the lowering requires the reference's
row-major linearization so every device array compares elementwise with the
reference's global vectors.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class GridShape:
    """Dimensions of a 2D or 3D pixel grid (grid.py:21-52)."""

    dims: tuple

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        if len(dims) not in (2, 3):
            raise ValueError(f"grid must be 2D or 3D, got {len(dims)} axes")
        if any(d < 1 for d in dims):
            raise ValueError(f"all grid dimensions must be positive, got {dims}")
        object.__setattr__(self, "dims", dims)

    @property
    def n(self) -> int:
        p = 1
        for d in self.dims:
            p *= d
        return p

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def strides(self) -> tuple:
        s = [1] * len(self.dims)
        for a in range(len(self.dims) - 2, -1, -1):
            s[a] = s[a + 1] * self.dims[a + 1]
        return tuple(s)


def index_of(shape: GridShape, coords) -> int:
    coords = tuple(int(c) for c in coords)
    if len(coords) != shape.ndim:
        raise ValueError(f"expected {shape.ndim} coordinates, got {len(coords)}")
    idx = 0
    for c, d, s in zip(coords, shape.dims, shape.strides):
        if not 0 <= c < d:
            raise ValueError(f"coordinate {coords} outside grid {shape.dims}")
        idx += c * s
    return idx


def coords_of(shape: GridShape, index: int) -> tuple:
    index = int(index)
    if not 0 <= index < shape.n:
        raise ValueError(f"index {index} outside grid of {shape.n} pixels")
    out = []
    for s in shape.strides:
        out.append(index // s)
        index %= s
    return tuple(out)
