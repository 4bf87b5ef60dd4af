"""Seeded synthetic tensors standing in for the BASELINE.json configs.

No public dataset is named for this path; these generators
draw tensors with the shapes, nonzero counts and value laws BASELINE.json
lists.  Coordinates are drawn per mode from a uniform law or a bounded Zipf
law P(i) ∝ (i+1)^-s on {0..I-1} (inverse-CDF sampling), and duplicate
coordinate tuples are *rejected* (first occurrence in draw order is kept)
until exactly `nnz` distinct tuples remain.  This differs on purpose from the
reference's `random_tensor` (pkg/src/altotensor/coo.py:211-230), which sums
collisions and returns fewer elements.

This module is host-side input generation (plumbing, never timed).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_TENSOR_BASE = 1000
SEED_FACTOR_BASE = 2000


@dataclass(frozen=True)
class SynthConfig:
    name: str
    dims: tuple[int, ...]
    nnz: int
    laws: tuple[tuple[str, float], ...]  # per mode: ("uniform", 0) | ("zipf", s)
    values: str                            # "uniform01" | "lognormal" | "uniform_pm1"
    value_dtype: str                       # "float64" | "float32"
    rank: int
    als_iters: int = 0
    note: str = ""


CONFIGS: dict[int, SynthConfig] = {
    1: SynthConfig("cfg1", (1000, 800, 600), 100_000,
                   (("uniform", 0),) * 3, "uniform01", "float64", 16, 5),
    2: SynthConfig("cfg2", (200_000, 150_000, 100_000), 50_000_000,
                   (("zipf", 1.1),) * 3, "uniform01", "float32", 16),
    3: SynthConfig("cfg3", (10_000_000, 5_000_000, 2_000, 500), 100_000_000,
                   (("zipf", 1.2), ("zipf", 1.2), ("uniform", 0), ("uniform", 0)),
                   "lognormal", "float32", 32),
    4: SynthConfig("cfg4", (1000, 1000, 1000, 100, 50), 20_000_000,
                   (("uniform", 0),) * 5, "uniform_pm1", "float32", 16),
    5: SynthConfig("cfg5", (40_000_000, 20_000_000, 1_000_000), 500_000_000,
                   (("zipf", 1.05),) * 3, "uniform01", "float32", 16, 10),
}


class _ZipfSampler:
    """Inverse-CDF sampler of the bounded law P(i) ∝ (i+1)^-s, i in [0, n)."""

    def __init__(self, n: int, s: float):
        w = np.arange(1, n + 1, dtype=np.float64)
        np.power(w, -s, out=w)
        np.cumsum(w, out=w)
        w /= w[-1]
        self.cdf = w
        self.n = n

    def draw(self, rng: np.random.Generator, size: int) -> np.ndarray:
        u = rng.random(size)
        idx = np.searchsorted(self.cdf, u, side="right")
        np.minimum(idx, self.n - 1, out=idx)
        return idx.astype(np.int64, copy=False)


def _pack(coords: np.ndarray, dims) -> tuple[np.ndarray, ...]:
    """Pack coordinate rows into one or two int64 columns (mixed radix)."""
    bits = [max((int(d) - 1).bit_length(), 0) for d in dims]
    cols = []
    cur = np.zeros(coords.shape[0], dtype=np.int64)
    used = 0
    for n, b in enumerate(bits):
        if used + b > 62:
            cols.append(cur)
            cur = np.zeros(coords.shape[0], dtype=np.int64)
            used = 0
        cur |= coords[:, n] << used
        used += b
    cols.append(cur)
    return tuple(cols)


def _first_occurrence(cols: tuple[np.ndarray, ...]) -> np.ndarray:
    """Indices of the first occurrence of each distinct packed tuple, ascending."""
    if len(cols) == 1:
        perm = np.argsort(cols[0], kind="stable")
        s = cols[0][perm]
        fresh = np.empty(s.shape[0], dtype=bool)
        if s.shape[0]:
            fresh[0] = True
            np.not_equal(s[1:], s[:-1], out=fresh[1:])
    else:
        perm = np.lexsort(tuple(cols))  # stable; last column primary
        fresh = np.empty(perm.shape[0], dtype=bool)
        if perm.shape[0]:
            fresh[0] = True
            diff = np.zeros(perm.shape[0] - 1, dtype=bool)
            for c in cols:
                sc = c[perm]
                diff |= sc[1:] != sc[:-1]
            fresh[1:] = diff
    first = perm[fresh]
    first.sort()
    return first


def draw_coords(dims, nnz: int, laws, rng: np.random.Generator) -> np.ndarray:
    """`nnz` distinct coordinate rows, duplicates rejected in draw order."""
    if nnz > math.prod(int(d) for d in dims):
        raise ValueError("nnz exceeds index space")
    samplers = [(_ZipfSampler(int(d), s) if law == "zipf" else None)
                for d, (law, s) in zip(dims, laws)]
    have = np.empty((0, len(dims)), dtype=np.int64)
    want = nnz
    factor = 1.05
    while True:
        extra = max(int((want - have.shape[0]) * factor), 1024)
        batch = np.empty((extra, len(dims)), dtype=np.int64)
        for n, d in enumerate(dims):
            if samplers[n] is None:
                batch[:, n] = rng.integers(0, int(d), size=extra, dtype=np.int64)
            else:
                batch[:, n] = samplers[n].draw(rng, extra)
        allc = np.concatenate([have, batch]) if have.shape[0] else batch
        first = _first_occurrence(_pack(allc, dims))
        have = allc[first]
        if have.shape[0] >= want:
            return np.ascontiguousarray(have[:want])
        factor = min(factor * 1.5, 4.0)


def draw_values(kind: str, m: int, rng: np.random.Generator) -> np.ndarray:
    if kind == "uniform01":
        return rng.random(m)
    if kind == "lognormal":
        return rng.lognormal(0.0, 1.0, m)
    if kind == "uniform_pm1":
        return rng.uniform(-1.0, 1.0, m)
    raise ValueError(kind)


@dataclass
class SynthTensor:
    config: SynthConfig
    coords: np.ndarray          # (nnz, N) int64
    values: np.ndarray          # (nnz,) value_dtype
    seed: int
    meta: dict = field(default_factory=dict)


def make_tensor(cfg: int | SynthConfig, nnz: int | None = None,
                seed: int | None = None) -> SynthTensor:
    """Draw the config's tensor (optionally at a reduced nnz, same laws)."""
    c = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    m = c.nnz if nnz is None else int(nnz)
    sd = (SEED_TENSOR_BASE + int(c.name[3:])) if seed is None else seed
    rng = np.random.default_rng(sd)
    coords = draw_coords(c.dims, m, c.laws, rng)
    vals = draw_values(c.values, m, rng).astype(c.value_dtype)
    return SynthTensor(c, coords, vals, sd)


def make_factors(dims, rank: int, dtype="float64", seed: int = 0) -> list[np.ndarray]:
    """MTTKRP factors: default_rng(seed).random((I_n, R)) per mode, in order."""
    rng = np.random.default_rng(seed)
    return [rng.random((int(d), rank)).astype(dtype) for d in dims]


def make_tensor_device(cfg: int | SynthConfig, nnz: int | None = None, seed: int | None = None, device="cuda"):
    """Same laws as make_tensor, drawn on the GPU with torch's generator (fast
    benchmark inputs; not bit-identical to the NumPy stream).  Distinct
    coordinate tuples are obtained by drawing, deduplicating with
    torch.unique and keeping a uniformly random subset of exactly `nnz`.
    Returns (coords (nnz, N) int64, values (nnz,) value_dtype) on `device`."""
    import torch

    c = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    m = c.nnz if nnz is None else int(nnz)
    sd = (SEED_TENSOR_BASE + int(c.name[3:])) if seed is None else seed
    g = torch.Generator(device=device)
    g.manual_seed(sd)
    bits = [max((int(d) - 1).bit_length(), 0) for d in c.dims]
    cdfs = []
    for d, (law, s) in zip(c.dims, c.laws):
        if law == "zipf":
            w = torch.arange(1, int(d) + 1, dtype=torch.float64, device=device).pow_(-s)
            w = torch.cumsum(w, 0)
            cdfs.append(w / w[-1])
        else:
            cdfs.append(None)

    def draw(k):
        cols = []
        for n, d in enumerate(c.dims):
            if cdfs[n] is None:
                cols.append(torch.randint(0, int(d), (k,), generator=g, device=device, dtype=torch.int64))
            else:
                u = torch.rand(k, generator=g, device=device, dtype=torch.float64)
                cols.append(torch.clamp(torch.searchsorted(cdfs[n], u, right=True), max=int(d) - 1))
        return torch.stack(cols, 1)

    def pack(x):
        # two int64 words (mixed radix), exact for <= 124 total bits
        hi = torch.zeros(x.shape[0], dtype=torch.int64, device=device)
        lo = torch.zeros_like(hi)
        used = 0
        for n, b in enumerate(bits):
            if used + b <= 62:
                lo |= x[:, n] << used
            else:
                hi = (hi << b) | x[:, n]
            used += b
        return hi, lo

    have = None
    factor = 1.1
    while True:
        need = m - (0 if have is None else have.shape[0])
        batch = draw(max(int(need * factor), 1024))
        allc = batch if have is None else torch.cat([have, batch])
        hi, lo = pack(allc)
        key = torch.stack([hi, lo], 1)
        _, inv = torch.unique(key, dim=0, return_inverse=True)
        first = torch.full((int(inv.max()) + 1,), allc.shape[0], dtype=torch.int64, device=device)
        first.scatter_reduce_(0, inv, torch.arange(allc.shape[0], device=device), reduce="amin")
        have = allc[first]
        del allc, key, inv, hi, lo
        if have.shape[0] >= m:
            sel = torch.randperm(have.shape[0], generator=g, device=device)[:m]
            coords = have[sel].contiguous()
            break
        factor = min(factor * 1.5, 4.0)
    if c.values == "uniform01":
        vals = torch.rand(m, generator=g, device=device, dtype=torch.float64)
    elif c.values == "lognormal":
        vals = torch.exp(torch.randn(m, generator=g, device=device, dtype=torch.float64))
    else:
        vals = torch.rand(m, generator=g, device=device, dtype=torch.float64) * 2.0 - 1.0
    return coords, vals.to(torch.float32 if c.value_dtype == "float32" else torch.float64)
