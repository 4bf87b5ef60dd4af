"""Device-resident ALTO tensors: build (K1+K2+K3), partition (K5), conflict
plans (host), boundary flags (K6).

Drop-in for pkg/src/altotensor/format.py.  An AltoTensor keeps its sorted
keys and values in B200 HBM; `.indices` / `.values` materialise host copies
only when asked for.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from .coo import CooTensor, coalesce
from .layout import (AltoLayout, build_masks, c_layout, delinearize_device,
                     device_tables, keys_to_device, keys_to_host,
                     linearize_device)


def _torch():
    import torch

    return torch


class AltoTensor:
    """Sparse tensor with sorted bit-interleaved keys (format.py:28-76).

    `indices` is (nnz, width // 64) uint64, least significant word first;
    `values` is float64 (the reference's dtype).  Device copies live in
    `keys` ((nnz, n_words) int64 raw bits) and `vals` (float32 or float64 —
    float32 storage is kept when the caller supplies float32 values; the
    upcast to the float64 `.values` view is exact).

    Like the reference's frozen dataclass, a tensor is immutable: transforms
    return new tensors.  Device torch inputs are adopted without a copy, so
    the caller must not modify them afterwards (per-mode plans cached on the
    tensor — mode streams, pull plans, row indexes — assume fixed contents).
    The mode-stream kernel's replicated hot-row partials are cached scratch
    that each call leaves zeroed; two concurrent MTTKRPs on the same tensor
    from different streams must not run the mode-stream kernel at the same
    time (the pull engine allocates its scratch per call).
    """

    def __init__(self, layout: AltoLayout, indices, values):
        torch = _torch()
        self.layout = layout
        if isinstance(indices, torch.Tensor):
            keys = indices.to(device=_lib.cuda_device(), dtype=torch.int64).contiguous()
            host_idx = None
        else:
            host_idx = np.ascontiguousarray(indices, dtype=np.uint64)
            if host_idx.ndim != 2 or host_idx.shape[1] != layout.n_words:
                raise ValueError(f"indices must have shape (nnz, {layout.n_words}), got {host_idx.shape}")
            keys = None
        if isinstance(values, torch.Tensor):
            vdt = torch.float32 if values.dtype == torch.float32 else torch.float64
            vals = values.to(device=_lib.cuda_device(), dtype=vdt).contiguous()
            host_val = None
        else:
            varr = np.asarray(values)
            host_val = np.ascontiguousarray(varr, dtype=np.float32 if varr.dtype == np.float32 else np.float64)
            vals = None
        nnz = int(keys.shape[0]) if keys is not None else int(host_idx.shape[0])
        if keys is not None and (keys.ndim != 2 or keys.shape[1] != layout.n_words):
            raise ValueError(f"indices must have shape (nnz, {layout.n_words}), got {tuple(keys.shape)}")
        nv = int(vals.shape[0]) if vals is not None else int(host_val.shape[0])
        vnd = vals.ndim if vals is not None else host_val.ndim
        if vnd != 1 or nv != nnz:
            raise ValueError("values length must match number of indices")
        if keys is None:
            keys = keys_to_device(host_idx)
        if vals is None:
            vals = torch.from_numpy(host_val).to(_lib.cuda_device())
        self.keys = keys
        self.vals = vals
        self._host_idx = host_idx
        self._host_val = None
        self._cache: dict = {}

    def __setattr__(self, name, value):
        if name in ("layout", "keys", "vals") and name in self.__dict__:
            raise AttributeError(f"AltoTensor.{name} is read-only")
        object.__setattr__(self, name, value)

    @property
    def nnz(self) -> int:
        return int(self.keys.shape[0])

    @property
    def dims(self) -> tuple[int, ...]:
        return self.layout.dims

    @property
    def value_dtype(self):
        return self.vals.dtype

    @property
    def indices(self) -> np.ndarray:
        if self._host_idx is None:
            object.__setattr__(self, "_host_idx", keys_to_host(self.keys))
        return self._host_idx

    @property
    def values(self) -> np.ndarray:
        if self._host_val is None:
            object.__setattr__(self, "_host_val", self.vals.double().cpu().numpy())
        return self._host_val

    def linear_at(self, row: int) -> int:
        w = self.keys[row].cpu().numpy().view(np.uint64)
        return sum(int(x) << (64 * i) for i, x in enumerate(w))

    def linear_positions(self) -> list[int]:
        idx = self.indices
        return [sum(int(idx[r, w]) << (64 * w) for w in range(idx.shape[1])) for r in range(idx.shape[0])]

    def to_coo(self) -> CooTensor:
        coords = delinearize_device(self.layout, self.keys, -1).cpu().numpy()
        return coalesce(self.layout.dims, coords, self.values.copy())


def _value_dtype(spec, default):
    torch = _torch()
    if spec is None:
        return default
    if spec in ("float32", np.float32, torch.float32):
        return torch.float32
    if spec in ("float64", np.float64, torch.float64, float):
        return torch.float64
    raise ValueError(f"unsupported value dtype {spec!r}")


def build_alto_device(layout: AltoLayout, coords_dev, vals_dev) -> AltoTensor:
    """K1 linearize + K2 radix sort (+payload) + K3 duplicate check, all on device."""
    torch = _torch()
    lib = _lib.load()
    m = int(coords_dev.shape[0])
    keys, bad = linearize_device(layout, coords_dev)
    vals = vals_dev.clone()
    ws_bytes = lib.alto_sort_workspace_bytes(m, layout.n_words, vals.element_size())
    ws = torch.empty(max(int(ws_bytes), 8), dtype=torch.uint8, device=keys.device)
    _lib.check(lib.alto_sort_pairs(keys.data_ptr(), vals.data_ptr(), m, layout.n_words, vals.element_size(),
                                   layout.total_bits, ws.data_ptr(), ws_bytes, _lib.stream_ptr()),
               "alto_sort_pairs")
    first = torch.empty(1, dtype=torch.int64, device=keys.device)
    _lib.check(lib.alto_find_duplicate(keys.data_ptr(), m, layout.n_words, first.data_ptr(), _lib.stream_ptr()),
               "alto_find_duplicate")
    flags = torch.stack([bad[0], first[0]]).cpu()
    if int(flags[0]) >= 0:
        raise ValueError("coordinates out of range for layout dims")
    if int(flags[1]) >= 0:
        raise ValueError("duplicate coordinates; coalesce the tensor first")
    return AltoTensor(layout, keys, vals)


def build_alto(tensor: CooTensor, layout: AltoLayout | None = None, *, dtype=None) -> AltoTensor:
    """Encode a coalesced coordinate tensor into sorted ALTO form (format.py:85-100).

    Extension: `dtype` ("float32"/"float64") selects the device value storage
    (default float64, as the reference).
    """
    torch = _torch()
    if layout is None:
        layout = build_masks(tensor.dims)
    elif layout.dims != tuple(tensor.dims):
        raise ValueError("layout dims do not match tensor dims")
    dev = _lib.cuda_device()
    vdt = _value_dtype(dtype, torch.float64)
    coords = torch.from_numpy(np.ascontiguousarray(tensor.coords, dtype=np.int64)).to(dev)
    vals = torch.from_numpy(np.ascontiguousarray(tensor.values)).to(device=dev, dtype=vdt)
    return build_alto_device(layout, coords, vals)


@dataclass(frozen=True)
class PartitionSet:
    """Contiguous equal-size slices of a sorted ALTO tensor (format.py:103-124)."""

    offsets: np.ndarray
    intervals: np.ndarray
    spans: tuple[tuple[int, int], ...]

    @property
    def count(self) -> int:
        return len(self.offsets) - 1


def partition_offsets(m: int, count: int) -> np.ndarray:
    """Element ranges of sizes differing by <= 1, larger first (format.py:136-140)."""
    q, r = divmod(m, count)
    sizes = np.where(np.arange(count) < r, q + 1, q).astype(np.int64)
    return np.concatenate([np.zeros(1, dtype=np.int64), np.cumsum(sizes)])


def partition(tensor: AltoTensor, count: int) -> PartitionSet:
    """Equal-nnz partitions with per-mode intervals and key spans (format.py:127-154).

    The interval/span pass (K5) runs on the device in one streaming decode.
    """
    torch = _torch()
    m = tensor.nnz
    if not 1 <= count <= max(m, 1):
        raise ValueError(f"partition count {count} not in [1, {max(m, 1)}]")
    lay = tensor.layout
    offsets = partition_offsets(m, count)
    dev = tensor.keys.device
    iv = torch.empty((count, lay.order, 2), dtype=torch.int64, device=dev)
    sp = torch.zeros((count, 2, lay.n_words), dtype=torch.int64, device=dev)
    lib = _lib.load()
    _lib.check(lib.alto_partition(c_layout(lay), device_tables(lay).data_ptr(), tensor.keys.data_ptr(), m, count,
                                  iv.data_ptr(), sp.data_ptr(), _lib.stream_ptr()), "alto_partition")
    intervals = iv.cpu().numpy()
    words = sp.cpu().numpy().view(np.uint64)
    sizes = np.diff(offsets)
    spans = []
    for l in range(count):
        if sizes[l] == 0:
            continue
        a = sum(int(words[l, 0, w]) << (64 * w) for w in range(lay.n_words))
        b = sum(int(words[l, 1, w]) << (64 * w) for w in range(lay.n_words))
        spans.append((a, b))
    return PartitionSet(offsets, intervals, tuple(spans))


class Strategy(enum.Enum):
    """Output synchronization strategy (format.py:157-161)."""

    BUFFERED = "buffered"
    ATOMIC = "atomic"


@dataclass(frozen=True)
class ConflictPlan:
    """Per-mode synchronization plan (format.py:164-193)."""

    mode: int
    strategy: Strategy
    reuse: float
    offsets: np.ndarray
    overlaps: tuple[tuple[tuple[int, int], ...], ...] | None
    flag_bit: int | None

    @property
    def count(self) -> int:
        return len(self.offsets) - 1


# Average output-row reuse above which partitions stage into private
# interval buffers (format.py:196).
REUSE_THRESHOLD = 4.0


def shared_ranges(mode_iv: np.ndarray) -> tuple[tuple[tuple[int, int], ...], ...]:
    """Per-partition ranges of its interval also covered by another partition.

    Same result as the reference's pairwise O(L^2) intersect-and-merge
    (format.py:234-246), computed by one coverage sweep: the points of
    partition l's interval that another interval covers are exactly the
    points with coverage >= 2, so overlaps[l] = (runs of coverage >= 2)
    clipped to [lo_l, hi_l].
    """
    lo = mode_iv[:, 0].astype(np.int64)
    hi = mode_iv[:, 1].astype(np.int64)
    live = lo <= hi
    if live.sum() < 2:
        return tuple(() for _ in range(len(lo)))
    pos = np.concatenate([lo[live], hi[live] + 1])
    delta = np.concatenate([np.ones(live.sum(), np.int64), -np.ones(live.sum(), np.int64)])
    order = np.argsort(pos, kind="stable")
    pos, delta = pos[order], delta[order]
    uniq, first = np.unique(pos, return_index=True)
    cover = np.cumsum(np.add.reduceat(delta, first))
    # coverage cover[k] holds on [uniq[k], uniq[k+1]-1]
    hot = np.nonzero(cover[:-1] >= 2)[0]
    runs_lo: list[int] = []
    runs_hi: list[int] = []
    for k in hot:
        a, b = int(uniq[k]), int(uniq[k + 1]) - 1
        if runs_hi and a == runs_hi[-1] + 1:
            runs_hi[-1] = b
        else:
            runs_lo.append(a)
            runs_hi.append(b)
    rl = np.asarray(runs_lo, dtype=np.int64)
    rh = np.asarray(runs_hi, dtype=np.int64)
    out = []
    for l in range(len(lo)):
        if not live[l] or rl.size == 0:
            out.append(())
            continue
        a = int(np.searchsorted(rh, lo[l], side="left"))
        b = int(np.searchsorted(rl, hi[l], side="right"))
        out.append(tuple((max(int(rl[k]), int(lo[l])), min(int(rh[k]), int(hi[l]))) for k in range(a, b)))
    return tuple(out)


def plan_conflicts(tensor: AltoTensor, parts: PartitionSet, mode: int,
                   force_strategy: Strategy | None = None) -> ConflictPlan:
    """Strategy choice and shared-row ranges (format.py:210-254); host logic."""
    order = tensor.layout.order
    if not 0 <= mode < order:
        raise ValueError(f"mode {mode} out of range for order {order}")
    reuse = tensor.nnz / tensor.layout.dims[mode]
    strategy = force_strategy
    if strategy is None:
        strategy = Strategy.BUFFERED if reuse > REUSE_THRESHOLD else Strategy.ATOMIC
    overlaps = None
    flag_bit = None
    if strategy is Strategy.ATOMIC:
        if tensor.layout.total_bits < tensor.layout.width:
            flag_bit = tensor.layout.total_bits
        overlaps = shared_ranges(np.asarray(parts.intervals)[:, mode, :])
    return ConflictPlan(mode, strategy, reuse, parts.offsets, overlaps, flag_bit)


def apply_boundary_flags(tensor: AltoTensor, plan: ConflictPlan) -> AltoTensor:
    """Copy with the flag bit set on shared-row elements (format.py:257-285), K6 on device."""
    torch = _torch()
    if plan.strategy is not Strategy.ATOMIC or plan.overlaps is None:
        raise ValueError("boundary flags only apply to atomic plans")
    if plan.flag_bit is None:
        raise ValueError("no unused index bit available for flags")
    if plan.offsets[-1] != tensor.nnz:
        raise ValueError("plan does not match tensor (element counts differ)")
    offs = np.asarray(plan.offsets, dtype=np.int64)
    count = len(offs) - 1
    if tensor.nnz == 0:
        return AltoTensor(tensor.layout, tensor.keys.clone(), tensor.vals)
    # any split of [0, nnz) the plan carries is accepted, as by the reference
    # (format.py:274-284 loops over plan.offsets); equal-size splits use the
    # closed form on device, others pass the offsets
    d_offs = None
    if not np.array_equal(offs, partition_offsets(tensor.nnz, count)):
        d_offs = torch.from_numpy(offs.copy()).to(tensor.keys.device)
    ptr = np.zeros(count + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(o) for o in plan.overlaps])
    flat = [r for o in plan.overlaps for r in o]
    lo = np.asarray([r[0] for r in flat] or [0], dtype=np.int64)
    hi = np.asarray([r[1] for r in flat] or [-1], dtype=np.int64)
    dev = tensor.keys.device
    d_ptr = torch.from_numpy(ptr).to(dev)
    d_lo = torch.from_numpy(lo).to(dev)
    d_hi = torch.from_numpy(hi).to(dev)
    out = torch.empty_like(tensor.keys)
    lib = _lib.load()
    lay = tensor.layout
    _lib.check(lib.alto_apply_flags(c_layout(lay), device_tables(lay).data_ptr(), tensor.keys.data_ptr(), tensor.nnz,
                                    count, plan.mode, plan.flag_bit, d_ptr.data_ptr(), d_lo.data_ptr(),
                                    d_hi.data_ptr(), None if d_offs is None else d_offs.data_ptr(), out.data_ptr(),
                                    _lib.stream_ptr()), "alto_apply_flags")
    return AltoTensor(lay, out, tensor.vals)


def read_flags_device(tensor: AltoTensor, flag_bit: int):
    torch = _torch()
    out = torch.empty(tensor.nnz, dtype=torch.uint8, device=tensor.keys.device)
    lib = _lib.load()
    _lib.check(lib.alto_read_flags(tensor.keys.data_ptr(), tensor.nnz, tensor.layout.n_words, int(flag_bit),
                                   out.data_ptr(), _lib.stream_ptr()), "alto_read_flags")
    return out


def read_flags(tensor: AltoTensor, flag_bit: int) -> np.ndarray:
    """Per-element flag bits as bool (format.py:288-291)."""
    return read_flags_device(tensor, flag_bit).cpu().numpy().astype(bool)


def clear_flags(tensor: AltoTensor, flag_bit: int) -> AltoTensor:
    """Copy with the flag bit cleared (format.py:294-299)."""
    torch = _torch()
    out = torch.empty_like(tensor.keys)
    lib = _lib.load()
    _lib.check(lib.alto_clear_flags(tensor.keys.data_ptr(), tensor.nnz, tensor.layout.n_words, int(flag_bit),
                                    out.data_ptr(), _lib.stream_ptr()), "alto_clear_flags")
    return AltoTensor(tensor.layout, out, tensor.vals)
