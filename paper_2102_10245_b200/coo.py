"""Coordinate-list input type (host).

Mirror of the reference's CooTensor (pkg/src/altotensor/coo.py:31-94), the
input of build_alto.  COO ingestion (coalesce, .tns parsing) is outside the
hot path; `coalesce` and `random_tensor` exist so
callers and tests can prepare inputs exactly as with the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np


@dataclass(frozen=True)
class CooTensor:
    """Sparse tensor as a coordinate list: dims, (nnz, order) int64 coords,
    (nnz,) float64 values (coo.py:31-67 validation rules)."""

    dims: tuple[int, ...]
    coords: np.ndarray
    values: np.ndarray

    def __post_init__(self) -> None:
        ext = tuple(int(d) for d in self.dims)
        if not ext:
            raise ValueError("tensor needs at least one mode")
        if min(ext) < 1:
            raise ValueError(f"dimensions must be positive, got {ext}")
        c = np.ascontiguousarray(self.coords, dtype=np.int64)
        v = np.ascontiguousarray(self.values, dtype=np.float64)
        if c.ndim != 2 or c.shape[1] != len(ext):
            raise ValueError(f"coords must have shape (nnz, {len(ext)}), got {c.shape}")
        if v.shape != (c.shape[0],):
            raise ValueError("values length must match number of coordinate rows")
        if c.size and (c.min() < 0 or (c >= np.asarray(ext, dtype=np.int64)).any()):
            raise ValueError("coordinates out of range for dims")
        object.__setattr__(self, "dims", ext)
        object.__setattr__(self, "coords", c)
        object.__setattr__(self, "values", v)

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.coords.shape[0])

    @property
    def density(self) -> float:
        return self.nnz / math.prod(self.dims)

    def coalesce(self) -> "CooTensor":
        return coalesce(self.dims, self.coords, self.values)

    def isequal(self, other: "CooTensor") -> bool:
        if self.dims != other.dims:
            return False
        a, b = self.coalesce(), other.coalesce()
        return bool(np.array_equal(a.coords, b.coords) and np.array_equal(a.values, b.values))


def coalesce(dims: Sequence[int], coords, values) -> CooTensor:
    """Rows sorted mode-0 major, duplicates summed (coo.py:97-114 semantics)."""
    c = np.ascontiguousarray(coords, dtype=np.int64)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if c.shape[0] == 0:
        return CooTensor(tuple(dims), c.reshape(0, len(dims)), v)
    order = np.lexsort(c.T[::-1])
    c = c[order]
    v = v[order]
    head = np.ones(c.shape[0], dtype=bool)
    head[1:] = (c[1:] != c[:-1]).any(axis=1)
    seg = np.cumsum(head) - 1
    return CooTensor(tuple(dims), c[head], np.bincount(seg, weights=v))


def random_tensor(dims: Sequence[int], target_nnz: int, seed: int) -> CooTensor:
    """Uniform coordinates and U[0,1) values, collisions summed (coo.py:211-230)."""
    ext = tuple(int(d) for d in dims)
    if any(d < 1 for d in ext):
        raise ValueError(f"dimensions must be positive, got {ext}")
    if target_nnz < 0:
        raise ValueError("target_nnz must be nonnegative")
    if target_nnz > math.prod(ext):
        raise ValueError(f"target_nnz {target_nnz} exceeds index space {math.prod(ext)}")
    rng = np.random.default_rng(seed)
    c = rng.integers(0, ext, size=(target_nnz, len(ext)), dtype=np.int64)
    v = rng.random(target_nnz)
    return coalesce(ext, c, v)
