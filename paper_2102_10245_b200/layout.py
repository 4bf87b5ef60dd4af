"""ALTO bit layout (host) and the device codecs (K1 linearize, K4 delinearize).

Drop-in for pkg/src/altotensor/layout.py.  The layout rule is O(total_bits)
host logic; every per-element encode/decode runs on the B200 through
libalto_b200.so (alto_linearize / alto_delinearize), including the scalar
helpers, so there is no host bit-twiddling path.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib

SUPPORTED_WIDTHS = (64, 128)
MAX_BITS = 128


class WidthOverflowError(ValueError):
    """More index bits than the widest storage word (layout.py:27-28)."""


def bits_for(dim: int) -> int:
    """ceil(log2 dim) index bits, 0 for extent 1 (layout.py:31-35)."""
    if dim < 1:
        raise ValueError(f"extent must be positive, got {dim}")
    return int(dim - 1).bit_length()


@dataclass(frozen=True)
class AltoLayout:
    """Bit layout of the linearized index (layout.py:38-71).

    positions[n][g] is the key bit holding bit g of mode n; masks[n] is the
    union of mode n's positions.
    """

    dims: tuple[int, ...]
    bits: tuple[int, ...]
    positions: tuple[tuple[int, ...], ...]
    masks: tuple[int, ...]
    total_bits: int
    width: int

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def n_words(self) -> int:
        return self.width // 64


def build_masks(dims: Sequence[int]) -> AltoLayout:
    """Adaptive interleaved layout (layout.py:74-102).

    Significance group g collects bit g of every mode that still has bits
    left; inside a group the modes are ordered by ascending extent, ties by
    mode number, and take consecutive key bits from the least significant
    free position upward.  Width is 64 when the total fits, else 128; more
    than 128 bits raises WidthOverflowError.
    """
    ext = tuple(int(d) for d in dims)
    if len(ext) == 0:
        raise ValueError("need at least one mode")
    nbits = tuple(bits_for(d) for d in ext)
    total = sum(nbits)
    if total > MAX_BITS:
        raise WidthOverflowError(f"shape {ext} needs {total} index bits, more than {MAX_BITS}")
    width = 64 if total <= 64 else 128
    rank_order = sorted(range(len(ext)), key=lambda n: (ext[n], n))
    slots: list[list[int]] = [[] for _ in ext]
    cursor = 0
    for g in range(max(nbits)):
        for n in rank_order:
            if nbits[n] > g:
                slots[n].append(cursor)
                cursor += 1
    masks = tuple(sum(1 << p for p in s) for s in slots)
    return AltoLayout(ext, nbits, tuple(tuple(s) for s in slots), masks, total, width)


# ---------------------------------------------------------------------------
# device-side helpers

_CLAYOUT_CACHE: dict = {}
_TABLE_CACHE: dict = {}


def c_layout(layout: AltoLayout) -> _lib.CLayout:
    """C struct for the ABI (cached per layout)."""
    c = _CLAYOUT_CACHE.get(layout)
    if c is None:
        if layout.order > _lib.ALTO_MAX_ORDER:
            raise ValueError(f"device path supports order <= {_lib.ALTO_MAX_ORDER}")
        c = _lib.CLayout()
        c.order = layout.order
        c.n_words = layout.n_words
        c.total_bits = layout.total_bits
        c.width = layout.width
        for n in range(layout.order):
            c.dims[n] = layout.dims[n]
            c.bits[n] = layout.bits[n]
            for g, p in enumerate(layout.positions[n]):
                c.pos[n][g] = p
        _CLAYOUT_CACHE[layout] = c
    return c


def device_tables(layout: AltoLayout):
    """Device encode/decode tables for the layout (cached per device)."""
    import torch

    dev = _lib.cuda_device()
    key = (layout, dev.index)
    t = _TABLE_CACHE.get(key)
    if t is None:
        lib = _lib.load()
        cl = c_layout(layout)
        nbytes = lib.alto_tables_bytes(cl)
        t = torch.empty(max(int(nbytes), 8), dtype=torch.uint8, device=dev)
        _lib.check(lib.alto_build_tables(cl, t.data_ptr(), _lib.stream_ptr()), "alto_build_tables")
        _TABLE_CACHE[key] = t
    return t


def _as_device(x, dtype):
    import torch

    dev = _lib.cuda_device()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(x)
    return torch.from_numpy(arr).to(device=dev, dtype=dtype).contiguous()


def keys_to_host(keys_dev) -> np.ndarray:
    """(M, n_words) int64 device tensor -> (M, n_words) uint64 numpy."""
    return keys_dev.cpu().numpy().view(np.uint64)


def keys_to_device(words) -> "object":
    """uint64 words (numpy or torch) -> (M, n_words) int64 device tensor (raw bits)."""
    import torch

    if isinstance(words, torch.Tensor):
        return words.to(device=_lib.cuda_device(), dtype=torch.int64).contiguous()
    w = np.ascontiguousarray(words)
    if w.dtype != np.uint64:
        w = w.astype(np.uint64)
    return torch.from_numpy(w.view(np.int64)).to(_lib.cuda_device()).contiguous()


def linearize_device(layout: AltoLayout, coords_dev):
    """K1 on device: (M, N) int64 device coords -> ((M, n_words) int64 keys, bad_row)."""
    import torch

    lib = _lib.load()
    m = int(coords_dev.shape[0])
    keys = torch.empty((m, layout.n_words), dtype=torch.int64, device=coords_dev.device)
    bad = torch.empty(1, dtype=torch.int64, device=coords_dev.device)
    tab = device_tables(layout)
    _lib.check(lib.alto_linearize(c_layout(layout), tab.data_ptr(), coords_dev.data_ptr(), m, keys.data_ptr(),
                                  bad.data_ptr(), _lib.stream_ptr()), "alto_linearize")
    return keys, bad


def delinearize_device(layout: AltoLayout, keys_dev, mode: int = -1):
    """K4 on device: keys -> (M, N) int64 (mode=-1) or (M,) int64 for one mode."""
    import torch

    lib = _lib.load()
    m = int(keys_dev.shape[0])
    shape = (m, layout.order) if mode < 0 else (m,)
    out = torch.empty(shape, dtype=torch.int64, device=keys_dev.device)
    tab = device_tables(layout)
    _lib.check(lib.alto_delinearize(c_layout(layout), tab.data_ptr(), keys_dev.data_ptr(), m, int(mode),
                                    out.data_ptr(), _lib.stream_ptr()), "alto_delinearize")
    return out


# ---------------------------------------------------------------------------
# reference API


def _coords_array(layout: AltoLayout, coords) -> np.ndarray:
    arr = np.ascontiguousarray(coords, dtype=np.int64)
    if arr.ndim != 2 or arr.shape[1] != layout.order:
        raise ValueError(f"coords must have shape (nnz, {layout.order}), got {arr.shape}")
    return arr


def linearize_array(layout: AltoLayout, coords) -> np.ndarray:
    """Encode coordinate rows (layout.py:148-160) on the device.

    Returns (nnz, width // 64) uint64, least significant word first.  A torch
    CUDA tensor input returns the device tensor (int64 storage, raw bits).
    """
    import torch

    if isinstance(coords, torch.Tensor):
        if coords.ndim != 2 or coords.shape[1] != layout.order:
            raise ValueError(f"coords must have shape (nnz, {layout.order}), got {tuple(coords.shape)}")
        keys, bad = linearize_device(layout, _as_device(coords, torch.int64))
        if int(bad.item()) >= 0:
            raise ValueError("coordinates out of range for layout dims")
        return keys
    arr = _coords_array(layout, coords)
    keys, bad = linearize_device(layout, _as_device(arr, torch.int64))
    if int(bad.item()) >= 0:
        raise ValueError("coordinates out of range for layout dims")
    return keys_to_host(keys)


def _words_array(layout: AltoLayout, words):
    import torch

    if isinstance(words, torch.Tensor):
        if words.ndim != 2 or words.shape[1] != layout.n_words:
            raise ValueError(f"index words must have shape (nnz, {layout.n_words}), got {tuple(words.shape)}")
        return keys_to_device(words), True
    w = np.ascontiguousarray(words, dtype=np.uint64)
    if w.ndim != 2 or w.shape[1] != layout.n_words:
        raise ValueError(f"index words must have shape (nnz, {layout.n_words}), got {w.shape}")
    return keys_to_device(w), False


def extract_mode_array(layout: AltoLayout, words, mode: int) -> np.ndarray:
    """One mode's coordinates as int64 (layout.py:163-169), decoded on device."""
    if not 0 <= mode < layout.order:
        raise ValueError(f"mode {mode} out of range for order {layout.order}")
    dev, is_torch = _words_array(layout, words)
    out = delinearize_device(layout, dev, mode)
    return out if is_torch else out.cpu().numpy()


def delinearize_array(layout: AltoLayout, words) -> np.ndarray:
    """(nnz, order) int64 coordinates (layout.py:172-182), decoded on device."""
    dev, is_torch = _words_array(layout, words)
    out = delinearize_device(layout, dev, -1)
    return out if is_torch else out.cpu().numpy()


def linearize(layout: AltoLayout, coords: Sequence[int]) -> int:
    """Encode one coordinate tuple (layout.py:105-116) — a 1-element device call."""
    if len(coords) != layout.order:
        raise ValueError(f"expected {layout.order} coordinates, got {len(coords)}")
    vals = [int(c) for c in coords]
    for n, c in enumerate(vals):
        if not 0 <= c < layout.dims[n]:
            raise ValueError(f"coordinate {c} out of range for mode {n}")
    words = linearize_array(layout, np.asarray([vals], dtype=np.int64))[0]
    return sum(int(w) << (64 * i) for i, w in enumerate(words))


def delinearize(layout: AltoLayout, pos: int) -> tuple[int, ...]:
    """Decode one linear index (layout.py:119-132) — a 1-element device call.

    Bits outside the storage width and above total_bits are ignored.
    """
    p = int(pos) & ((1 << layout.width) - 1)
    words = np.asarray([[(p >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(layout.n_words)]], dtype=np.uint64)
    row = delinearize_array(layout, words)[0]
    return tuple(int(c) for c in row)
