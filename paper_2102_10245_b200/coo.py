"""Coordinate-list input type and COO ingestion.

Mirror of the reference's CooTensor (pkg/src/altotensor/coo.py:31-94), the
input of build_alto, plus the ingestion in front of it: `coalesce` (sort +
duplicate sums) runs on the device (alto_coalesce, bitwise equal to the
reference's lexsort + bincount), `parse_tns` / `write_tns` are the text
format (coo.py:117-208), `random_tensor` the reference's sampler.
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


def _bits_for(d: int) -> int:
    return max((int(d) - 1).bit_length(), 0)


def coalesce_device(dims: Sequence[int], coords, values):
    """Device coalesce (alto_coalesce): (coords (k, N) int64, values (k,)
    float64) device tensors, rows sorted mode-0 major, duplicates summed in
    float64 in stable order (bitwise equal to coo.py:97-114's bincount)."""
    import ctypes

    import torch

    from . import _lib

    dev = _lib.cuda_device()
    c = torch.as_tensor(coords, dtype=torch.int64).to(dev).contiguous()
    v = torch.as_tensor(values, dtype=torch.float64).to(dev).contiguous()
    m, order = int(c.shape[0]), len(dims)
    c = c.reshape(m, order)
    bits = (ctypes.c_int32 * order)(*[_bits_for(d) for d in dims])
    nw = 2 if sum(bits) > 64 else 1
    lib = _lib.load()
    wsb = int(lib.alto_coalesce_workspace_bytes(m, nw))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    oc = torch.empty((m, order), dtype=torch.int64, device=dev)
    ov = torch.empty(m, dtype=torch.float64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(lib.alto_coalesce(c.data_ptr(), v.data_ptr(), m, order, bits, oc.data_ptr(), ov.data_ptr(),
                                 cnt.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr()), "alto_coalesce")
    k = int(cnt.item())
    return oc[:k], ov[:k]


def coalesce(dims: Sequence[int], coords, values) -> CooTensor:
    """Rows sorted mode-0 major, duplicates summed (coo.py:97-114), on the device."""
    c = np.ascontiguousarray(coords, dtype=np.int64).reshape(-1, len(dims))
    if c.shape[0] == 0:
        return CooTensor(tuple(dims), c, np.ascontiguousarray(values, dtype=np.float64))
    oc, ov = coalesce_device(dims, c, values)
    return CooTensor(tuple(dims), oc.cpu().numpy(), ov.cpu().numpy())


class TnsParseError(ValueError):
    """Raised when tensor text input is malformed (coo.py:27-28)."""


def _lines(source):
    if isinstance(source, str):
        return source.splitlines()
    return source


def parse_tns(source, dims: Sequence[int] | None = None) -> CooTensor:
    """FROSTT-style text (coo.py:117-189) -> coalesced CooTensor: one element
    per line (N one-based indices, then the value), blank lines and `#`
    comments skipped, an optional `# dims: I1 I2 ...` comment before the first
    data line (the `dims` argument wins), extents otherwise from the maxima.
    Text is tokenised on the host; the coalesce (sort + duplicate sums) runs
    on the device."""
    idx_rows: list[list[str]] = []
    val_tok: list[str] = []
    linenos: list[int] = []
    header = None
    order = None
    for lineno, raw in enumerate(_lines(source), start=1):
        text = raw.strip()
        if not text:
            continue
        if text[0] == "#":
            body = text[1:].strip()
            if order is None and header is None and body.startswith("dims:"):
                try:
                    header = tuple(int(x) for x in body[5:].split())
                except ValueError:
                    raise TnsParseError(f"line {lineno}: malformed dims header {text!r}") from None
                if not header or min(header) < 1:
                    raise TnsParseError(f"line {lineno}: dims header needs positive extents")
            continue
        tok = text.split()
        if order is None:
            order = len(tok) - 1
            if order < 1:
                raise TnsParseError(f"line {lineno}: expected at least one index and a value")
        if len(tok) != order + 1:
            raise TnsParseError(f"line {lineno}: expected {order + 1} fields, got {len(tok)}")
        idx_rows.append(tok[:-1])
        val_tok.append(tok[-1])
        linenos.append(lineno)
    # numeric conversion per line, so errors name the offending line
    rows = np.empty((len(idx_rows), order or 0), dtype=np.int64)
    vals = np.empty(len(val_tok), dtype=np.float64)
    for r, (it, vt, ln) in enumerate(zip(idx_rows, val_tok, linenos)):
        try:
            rows[r] = [int(x) for x in it]
            vals[r] = float(vt)
        except (ValueError, OverflowError):
            raise TnsParseError(f"line {ln}: malformed entry {' '.join(it + [vt])!r}") from None
        lo = int(rows[r].min())
        if lo < 1:
            raise TnsParseError(f"line {ln}: indices are one-based, got {lo}")
    if dims is None:
        dims = header
    if order is None:
        if dims is None:
            raise TnsParseError("no data lines found")
        order = len(dims)
        rows = rows.reshape(0, order)
    coords = rows - 1
    if dims is None:
        shape = tuple(int(x) + 1 for x in coords.max(axis=0))
    else:
        shape = tuple(int(x) for x in dims)
        if len(shape) != order:
            raise TnsParseError(f"declared {len(shape)} dimensions but data has {order} modes")
        if coords.size and (coords >= np.asarray(shape, dtype=np.int64)).any():
            raise TnsParseError("coordinate exceeds declared dimensions")
    return coalesce(shape, coords, vals)


def write_tns(tensor: CooTensor, stream=None):
    """One line per element, one-based indices, `# dims:` header, values via
    repr (exact round trip) (coo.py:192-208).  Returns the text if no stream."""
    lines = ["# dims: " + " ".join(str(d) for d in tensor.dims)]
    lines += [" ".join([str(int(i) + 1) for i in row] + [repr(float(v))])
              for row, v in zip(tensor.coords, tensor.values)]
    text = "\n".join(lines) + "\n"
    if stream is None:
        return text
    stream.write(text)
    return None


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
