"""MTTKRP on the B200: drop-in for pkg/src/altotensor/mttkrp.py.

Engines (all device code in libalto_b200.so):
  * streaming tile kernel (`mttkrp_stream`, alto_mttkrp) — the fast path:
    per-CTA interval buffers in shared memory with a float64 merge, or
    float64 atomics for wide tiles.  Used for Atomic plans (like the
    reference's atomic path it is not bitwise reproducible across runs).
  * exact-order engine (`mttkrp_exact`, alto_mttkrp_exact) — deterministic:
    per-row sums in element order, split at partition boundaries and merged
    in ascending partition order, in float64.  This is exactly the
    arithmetic order of mttkrp_seq (mttkrp.py:108-117) and of the Buffered
    stage + pull (mttkrp.py:148-172), so results are bitwise equal to the
    reference on float64 inputs and independent of `workers`.
  * COO kernel (`mttkrp_oracle`) over a coordinate list.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _lib
from .coo import CooTensor
from .format import (AltoTensor, ConflictPlan, PartitionSet, Strategy,
                     apply_boundary_flags, partition, plan_conflicts,
                     read_flags_device)
from .layout import c_layout, device_tables

# The reference's host chunk size (mttkrp.py:39); kept for API parity.
CHUNK = 1 << 17
# Elements per CTA tile of the streaming kernel.
DEFAULT_TILE = 1024
# float32 data with a float64 result: merge in float32 and upcast once.
F32_ACCUMULATE = __import__("os").environ.get("ALTO_F32_ACCUMULATE", "1") == "1"
# Streaming-kernel tuning switches (ALTO_STREAM_* in include/alto_b200.h).
STREAM_FLAGS = int(__import__("os").environ.get("ALTO_STREAM_FLAGS", "0"))


def _torch():
    import torch

    return torch


def _is_torch(x) -> bool:
    torch = _torch()
    return isinstance(x, torch.Tensor)


def _check_factors(dims: Sequence[int], factors, mode: int) -> int:
    """Shape validation with the reference's messages (mttkrp.py:42-61)."""
    if not 0 <= mode < len(dims):
        raise ValueError(f"mode {mode} out of range for order {len(dims)}")
    if len(factors) != len(dims):
        raise ValueError(f"expected {len(dims)} factor matrices, got {len(factors)}")
    rank = None
    for n, f in enumerate(factors):
        if f.ndim != 2:
            raise ValueError(f"factor {n} must be 2-D, got {f.ndim}-D")
        if f.shape[0] != dims[n]:
            raise ValueError(f"factor {n} has {f.shape[0]} rows, mode extent is {dims[n]}")
        if rank is None:
            rank = f.shape[1]
        elif f.shape[1] != rank:
            raise ValueError("factor matrices must share one rank")
    return int(rank)


_COPY_STREAM = {}


def _copy_stream(dev):
    """Side stream for host->device factor copies (one per device)."""
    torch = _torch()
    st = _COPY_STREAM.get(dev)
    if st is None:
        st = torch.cuda.Stream(device=dev)
        _COPY_STREAM[dev] = st
    return st


def factors_to_device(factors, dtype=None, skip: int | None = None) -> list:
    """Factors as contiguous device tensors (float64 unless dtype/torch input
    says otherwise).  `skip`: a host factor the MTTKRP of that mode never
    reads (the output mode's) is not copied; a 1-row placeholder of the same
    dtype and rank stands in for it.  Pinned host torch tensors are copied
    asynchronously on a side stream that the current stream then waits for,
    so a caller's next upload overlaps the previous call's kernels (as with
    any non_blocking copy, a pinned input must not be modified until the
    stream is synchronized)."""
    torch = _torch()
    dev = _lib.cuda_device()
    out = []
    cur = None
    for n, f in enumerate(factors):
        if (isinstance(f, torch.Tensor) and not f.is_cuda and f.is_pinned() and n != skip
                and (dtype is None or f.dtype == dtype) and f.is_contiguous()):
            if cur is None:
                cur = torch.cuda.current_stream(dev)
                side = _copy_stream(dev)
            with torch.cuda.stream(side):
                d = torch.empty(f.shape, dtype=f.dtype, device=dev)  # side-stream memory pool
                d.copy_(f, non_blocking=True)
            d.record_stream(cur)  # not reused before the work queued on `cur` that reads it
            out.append(d)
            continue
        if n == skip and not (isinstance(f, torch.Tensor) and f.is_cuda):
            a = f if isinstance(f, torch.Tensor) else np.asarray(f)
            is32 = (a.dtype == torch.float32) if isinstance(a, torch.Tensor) else (a.dtype == np.float32)
            dt = dtype or (torch.float32 if is32 else torch.float64)
            out.append(torch.zeros((1, int(a.shape[1])), dtype=dt, device=dev))
            continue
        if isinstance(f, torch.Tensor):
            dt = dtype or (torch.float32 if f.dtype == torch.float32 else torch.float64)
            out.append(f.to(device=dev, dtype=dt).contiguous())
        else:
            a = np.asarray(f)
            dt = dtype or (torch.float32 if a.dtype == np.float32 else torch.float64)
            out.append(torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dt).contiguous())
    if cur is not None:
        cur.wait_stream(_copy_stream(dev))
    return out


def _dt_code(t) -> int:
    torch = _torch()
    return _lib.ALTO_F32 if t.dtype == torch.float32 else _lib.ALTO_F64


def _args(tensor: AltoTensor, fdev: list, mode: int, out, tile: int = 0, zero_out: int = 1, vals=None):
    lay = tensor.layout
    vals = tensor.vals if vals is None else vals
    a = _lib.CMttkrpArgs()
    cl = c_layout(lay)
    a.lay = ctypes.pointer(cl)
    a.d_tables = device_tables(lay).data_ptr()
    a.keys = tensor.keys.data_ptr()
    a.values = vals.data_ptr()
    a.m = tensor.nnz
    a.mode = mode
    a.rank = int(fdev[0].shape[1])
    a.value_dtype = _dt_code(vals)
    fdt = {_dt_code(f) for f in fdev}
    if len(fdt) != 1:
        raise ValueError("factor matrices must share one dtype")
    a.factor_dtype = fdt.pop()
    for n, f in enumerate(fdev):
        a.factors[n] = f.data_ptr()
    a.out = out.data_ptr()
    a.out_dtype = _dt_code(out)
    a.tile = tile
    a.zero_out = zero_out
    a.n_hot = 0
    a.flags = STREAM_FLAGS
    a.fixed_scale = None
    a.packed = None
    a.pos = None
    a.plan = None
    a.cache_k = 0
    a.cache_modes = 0
    return a, cl


# Hot-row plan: rows holding more than HOT_TAU elements appear in almost every
# tile; their tile partials go to HOT_COPIES replicated buffers instead of
# contending on one L2 line (see alto_mttkrp_args in include/alto_b200.h).
HOT_TAU = 1024
HOT_MAX = 32768
# float32 copies take fewer adds each (precision); float64 copies fewer bytes
HOT_COPIES = {4: 64, 8: 32}


def hot_slots(tensor: AltoTensor, mode: int):
    """Per-mode hot-row slots (rows with more than HOT_TAU elements), cached:
    (slot map (I_mode,) int32, hot row ids, count) or None."""
    torch = _torch()
    key = ("hotslots", mode)
    if key in tensor._cache:
        return tensor._cache[key]
    res = None
    if tensor.nnz > HOT_TAU:
        lib = _lib.load()
        dim = tensor.layout.dims[mode]
        dev = tensor.keys.device
        _perm, ptr = row_index(tensor, mode)
        slot = torch.empty(dim, dtype=torch.int32, device=dev)
        kk = min(HOT_MAX, dim)
        rows = torch.empty(kk, dtype=torch.int32, device=dev)
        nhot = torch.zeros(1, dtype=torch.int32, device=dev)
        wsb = lib.alto_topk_rows_workspace_bytes(dim)
        ws = torch.empty(int(wsb), dtype=torch.uint8, device=dev)
        # the HOT_MAX rows with the most elements, if above HOT_TAU (hottest first)
        _lib.check(lib.alto_hot_rows(ptr.data_ptr(), dim, kk, HOT_TAU, rows.data_ptr(), slot.data_ptr(),
                                     nhot.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr()), "alto_hot_rows")
        n = int(nhot.item())
        if n > 0:
            res = (slot, rows, n)
    tensor._cache[key] = res
    return res


def hot_plan(tensor: AltoTensor, mode: int, rank: int, out_dtype=None):
    """Hot-row plan of one mode with zeroed replicated copies for (rank, output dtype), cached."""
    torch = _torch()
    out_dtype = out_dtype or torch.float64
    key = ("hot", mode, rank, out_dtype)
    if key in tensor._cache:
        return tensor._cache[key]
    hs = hot_slots(tensor, mode)
    plan = None
    if hs is not None:
        slot, rows, n = hs
        copies = HOT_COPIES[torch.empty(0, dtype=out_dtype).element_size()]
        buf = torch.zeros(copies * n * rank, dtype=out_dtype, device=tensor.keys.device)
        plan = (slot, rows, n, copies, buf)
    tensor._cache[key] = plan
    return plan


# Mode-stream hot plan: at most HOT_BOUND merges per replicated copy of a hot
# row (bounds same-address contention and float32 rounding of the copies),
# at most 2^HOT_MAX_LG copies per row.
HOT_BOUND = 1024
HOT_MAX_LG = 10


def hot_plan_ms(tensor: AltoTensor, mode: int, rank: int, out_dtype):
    """Hot-row plan of the mode-stream kernel (alto_hot_copies), cached:
    (hot_code (I_mode,) int32, hot rows, count, hot_base (count+1,) int32, zeroed copies) or None."""
    torch = _torch()
    T = ms_tile(tensor)
    key = ("hotms", mode, rank, out_dtype, T, MS_ORDER)
    if key in tensor._cache:
        return tensor._cache[key]
    hs = hot_slots(tensor, mode)
    plan = None
    if hs is not None:
        _slot, rows, n = hs
        dev = tensor.keys.device
        _perm, ptr = row_index(tensor, mode)
        code = torch.full((tensor.layout.dims[mode],), -1, dtype=torch.int32, device=dev)
        base = torch.empty(n + 1, dtype=torch.int32, device=dev)
        _lib.check(_lib.load().alto_hot_copies(ptr.data_ptr(), rows.data_ptr(), n, tensor.nnz, T, MS_ORDER, HOT_BOUND,
                                               HOT_MAX_LG, code.data_ptr(), base.data_ptr(), _lib.stream_ptr()),
                   "alto_hot_copies")
        total = int(base[n].item())
        buf = torch.zeros(total * rank, dtype=out_dtype, device=dev)
        plan = (code, rows, n, base, buf)
    tensor._cache[key] = plan
    return plan


def _set_hot(a, tensor: AltoTensor, mode: int, rank: int, out_dtype, ms) -> None:
    """Fill the hot-row plan fields of an alto_mttkrp_args for the kernel that will run."""
    if ms is not None:
        hp = hot_plan_ms(tensor, mode, rank, out_dtype)
        if hp is not None:
            code, rows, n, base, buf = hp
            a.hot_slot, a.hot_rows, a.n_hot, a.hot_copies, a.hot_buf, a.hot_base = (
                code.data_ptr(), rows.data_ptr(), n, 1, buf.data_ptr(), base.data_ptr())
        return
    hp = hot_plan(tensor, mode, rank, out_dtype)
    if hp is not None:
        slot, rows, n, copies, buf = hp
        a.hot_slot, a.hot_rows, a.n_hot, a.hot_copies, a.hot_buf = (slot.data_ptr(), rows.data_ptr(), n, copies,
                                                                   buf.data_ptr())


# Shared-memory budget (bytes per CTA) for the hot-input row cache.
CACHE_BUDGET = int(__import__("os").environ.get("ALTO_CACHE_BUDGET", 32 * 1024))
# Default planned variant: "plan2" (plan words + hot-input cache) or "pos".
PLAN_VARIANT = __import__("os").environ.get("ALTO_PLAN", "pos")


def topk_rows(tensor: AltoTensor, mode: int, k: int):
    """The k rows of `mode` with the most elements: (rows (k,) int32, slot map (I,) int32), cached."""
    torch = _torch()
    key = ("topk", mode, k)
    hit = tensor._cache.get(key)
    if hit is None:
        lib = _lib.load()
        dim = tensor.layout.dims[mode]
        dev = tensor.keys.device
        _perm, ptr = row_index(tensor, mode)
        rows = torch.empty(k, dtype=torch.int32, device=dev)
        smap = torch.empty(dim, dtype=torch.int32, device=dev)
        wsb = lib.alto_topk_rows_workspace_bytes(dim)
        ws = torch.empty(int(wsb), dtype=torch.uint8, device=dev)
        _lib.check(lib.alto_topk_rows(ptr.data_ptr(), dim, k, rows.data_ptr(), smap.data_ptr(), ws.data_ptr(), wsb,
                                      _lib.stream_ptr()), "alto_topk_rows")
        hit = (rows, smap)
        tensor._cache[key] = hit
    return hit


def stream_plan(tensor: AltoTensor, mode: int, rank: int, fbytes: int):
    """Per-mode plan words (alto_stream_plan) + hot-input row caches, cached."""
    torch = _torch()
    order = tensor.layout.order
    n_cache = min(order - 1, 3)
    k = max(0, min(255, CACHE_BUDGET // max(1, n_cache * rank * fbytes)))
    key = ("plan2", mode, k)
    hit = tensor._cache.get(key)
    if hit is not None:
        return hit
    lib = _lib.load()
    in_modes = [n for n in range(order) if n != mode][:n_cache]
    cache_rows, smaps = [], [None] * order
    if k > 0:
        for n in in_modes:
            rows, smap = topk_rows(tensor, n, k)
            cache_rows.append(rows)
            smaps[n] = smap
    hs = hot_slots(tensor, mode)
    plan = torch.empty(max(tensor.nnz, 1), dtype=torch.int64, device=tensor.keys.device)
    arr = (ctypes.c_void_p * order)(*[None if sm is None else sm.data_ptr() for sm in smaps])
    _lib.check(lib.alto_stream_plan(c_layout(tensor.layout), packed_keys(tensor).data_ptr(), tensor.nnz, mode, arr,
                                    None if hs is None else hs[0].data_ptr(), plan.data_ptr(), _lib.stream_ptr()),
               "alto_stream_plan")
    hit = {"plan": plan, "cache_rows": cache_rows, "k": k if cache_rows else 0, "modes": len(cache_rows)}
    tensor._cache[key] = hit
    return hit


# Per-mode stream tile length (elements); 0 disables the mode-stream kernel.
MS_TILE = int(__import__("os").environ.get("ALTO_MS_TILE", 1024))
# Mode-stream order: 1 (default) = the whole stream sorted by the mode's
# coordinate, ALTO order kept within a row (ALTO_MS_ROW_MAJOR); 0 = each tile
# (a contiguous ALTO key range) sorted by it.
MS_ORDER = int(__import__("os").environ.get("ALTO_MS_ORDER", 1))
# Lane groups take round-robin positions of a tile (1, default: the 8 elements
# of one warp instruction are consecutive, so their ALTO-ordered input rows
# share lines more often) or contiguous slices (0).
MS_RR = int(__import__("os").environ.get("ALTO_MS_RR", 1))


def ms_tile(tensor: AltoTensor) -> int:
    """Tile length of the tensor's mode streams: MS_TILE, halved (down to 128)
    for small tensors so that there are >= ~4 tiles per resident warp
    (148 SMs x 24 warps)."""
    t = MS_TILE
    while t > 128 and tensor.nnz < 148 * 24 * 4 * t:
        t //= 2
    return t


def mode_stream(tensor: AltoTensor, mode: int, vals=None):
    """Per-mode stream of the MTTKRP (alto_mode_stream), cached per (mode,
    value dtype): the ALTO stream in tiles of MS_TILE elements, each stably
    sorted by its `mode` coordinate, with hot-row flags.  -> (keys, values, tile)."""
    torch = _torch()
    vals = tensor.vals if vals is None else vals
    T = ms_tile(tensor)
    key = ("mstream", mode, vals.dtype, T, MS_ORDER, MS_RR)
    hit = tensor._cache.get(key)
    if hit is None:
        lib = _lib.load()
        lay = tensor.layout
        m = tensor.nnz
        dev = tensor.keys.device
        hs = hot_slots(tensor, mode)
        hot = hs is not None and lay.total_bits < 64 * lay.n_words
        ntiles = (m + T - 1) // T
        skeys = torch.empty((max(ntiles * T, 1), lay.n_words), dtype=tensor.keys.dtype, device=dev)
        svals = torch.empty(max(ntiles * T, 1), dtype=vals.dtype, device=dev)
        wsb = int(lib.alto_mode_stream_workspace_bytes(m))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        rc = lib.alto_mode_stream(c_layout(lay), packed_keys(tensor).data_ptr(), vals.data_ptr(), _dt_code(vals), m,
                                  mode, T, MS_ORDER | (4 if MS_RR else 0), hs[0].data_ptr() if hot else None,
                                  skeys.data_ptr(),
                                  svals.data_ptr(),
                                  ws.data_ptr(), wsb, _lib.stream_ptr())
        del ws
        if rc == _lib.ALTO_EUNSUPPORTED:
            hit = False  # field layout does not fit the key width: planned kernel instead
        else:
            _lib.check(rc, "alto_mode_stream")
            hit = (skeys, svals, T, MS_RR)
        tensor._cache[key] = hit
    return hit or None


def _set_stream(a, ms) -> None:
    sk, sv, st, rr = ms
    a.mkeys, a.mvals, a.mtile, a.mrr = sk.data_ptr(), sv.data_ptr(), st, 1 if rr else 0


# Ranks served by the mode-stream kernel (rank 32 stays on the planned kernel
# unless listed: it measured no faster on cfg3).
MS_RANKS = tuple(int(x) for x in __import__("os").environ.get("ALTO_MS_RANKS", "16").split(",") if x)


# Paired input modes (orders 4-5, float32, rank 16): two input modes whose
# row-wise product table (I_a * I_b rows) stays within MS_PAIR_BYTES are
# gathered as one row, so one gather replaces two (0 disables pairing).
MS_PAIR_BYTES = int(__import__("os").environ.get("ALTO_MS_PAIR_BYTES", 64 << 20))


def ms_pairs(dims, mode: int, rank: int, fbytes: int = 4, limit: int | None = None):
    """Input-mode pairs for the mode-stream kernel: the two smallest input
    modes, then the next two, while each pair's product table fits `limit`
    bytes (at most 2 pairs; orders 4-5, rank 16, float32 only)."""
    limit = MS_PAIR_BYTES if limit is None else limit
    if limit <= 0 or rank != 16 or fbytes != 4 or not 4 <= len(dims) <= 5:
        return []
    ins = sorted((n for n in range(len(dims)) if n != mode), key=lambda n: (dims[n], n))
    pairs = []
    for i in range(0, len(ins) - 1, 2):
        a, b = ins[i], ins[i + 1]
        if dims[a] * dims[b] * rank * fbytes > min(limit, (1 << 32) - 1):
            break
        pairs.append((a, b))
    return pairs


def _set_pairs(a, tensor: AltoTensor, fdev: list, mode: int, keep: list) -> None:
    """Build the product tables of the paired input modes (alto_krp_pair) and
    hand them to the mode-stream kernel."""
    torch = _torch()
    rank = int(fdev[0].shape[1])
    if tensor.vals.dtype != torch.float32 or fdev[0].dtype != torch.float32:
        return
    pairs = ms_pairs(tensor.layout.dims, mode, rank, 4)
    if not pairs:
        return
    lib = _lib.load()
    for i, (pa, pb) in enumerate(pairs):
        da, db = tensor.layout.dims[pa], tensor.layout.dims[pb]
        tab = torch.empty((da * db, rank), dtype=torch.float32, device=fdev[0].device)
        _lib.check(lib.alto_krp_pair(fdev[pa].data_ptr(), da, fdev[pb].data_ptr(), db, rank, _lib.ALTO_F32,
                                     tab.data_ptr(), _lib.stream_ptr()), "alto_krp_pair")
        keep.append(tab)
        a.pair_a[i], a.pair_b[i], a.pair_tab[i] = pa, pb, tab.data_ptr()
    a.n_pairs = len(pairs)


def _use_mode_stream(tensor: AltoTensor, rank: int, fbytes: int = 4) -> bool:
    """Mode-stream kernel for the ranks in MS_RANKS."""
    lay = tensor.layout
    return (MS_TILE > 0 and tensor.nnz > 0 and rank in MS_RANKS and 3 <= lay.order <= 5 and max(lay.bits) <= 31
            and tensor.nnz < (1 << 32) - 1 and max(lay.dims) * rank * fbytes < (1 << 32))


def packed_keys(tensor: AltoTensor):
    """Mode-contiguous re-encoding of the sorted keys (alto_pack_keys), cached."""
    torch = _torch()
    hit = tensor._cache.get("packed")
    if hit is None:
        lay = tensor.layout
        hit = torch.empty_like(tensor.keys)
        _lib.check(_lib.load().alto_pack_keys(c_layout(lay), device_tables(lay).data_ptr(), tensor.keys.data_ptr(),
                                              tensor.nnz, hit.data_ptr(), _lib.stream_ptr()), "alto_pack_keys")
        tensor._cache["packed"] = hit
    return hit


def subtile_order(tensor: AltoTensor, mode: int):
    """Per-mode row-sorted slot of each element in its 128-element sub-tile, cached."""
    torch = _torch()
    key = ("pos", mode)
    hit = tensor._cache.get(key)
    if hit is None:
        hit = torch.empty(max(tensor.nnz, 1), dtype=torch.uint8, device=tensor.keys.device)
        _lib.check(_lib.load().alto_subtile_order(c_layout(tensor.layout), packed_keys(tensor).data_ptr(), tensor.nnz,
                                                  mode, hit.data_ptr(), _lib.stream_ptr()), "alto_subtile_order")
        tensor._cache[key] = hit
    return hit


def mttkrp_stream(tensor: AltoTensor, fdev: list, mode: int, out=None, tile: int = DEFAULT_TILE,
                  zero_out: bool = True, hot: bool = True, out_dtype=None, planned: bool = True):
    """Fast streaming ALTO MTTKRP on device tensors -> (I_mode, R) device tensor
    (float64 by default; float32 when requested for float32 data/factors)."""
    torch = _torch()
    rank = int(fdev[0].shape[1])
    dim = tensor.layout.dims[mode]
    if tensor.vals.dtype == torch.float64 and fdev[0].dtype == torch.float32:
        fdev = [f.double() for f in fdev]  # exact upcast; the kernel pairs f64 values with f64 factors
    if out is None:
        out = torch.empty((dim, rank), dtype=out_dtype or torch.float64, device=tensor.keys.device)
    if (out.dtype == torch.float64 and tensor.vals.dtype == torch.float32 and fdev[0].dtype == torch.float32
            and F32_ACCUMULATE):
        # float32 data: accumulate with float32 merges (RED.F32x4; hot rows
        # still summed in float64 across copies), then upcast the result
        tmp = mttkrp_stream(tensor, fdev, mode, None, tile, True, hot, torch.float32, planned)
        if not zero_out:
            tmp64 = torch.empty_like(out)
            _lib.check(_lib.load().alto_cast_f32_f64(tmp.data_ptr(), tmp64.data_ptr(), tmp.numel(),
                                                     _lib.stream_ptr()), "alto_cast_f32_f64")
            out += tmp64
        else:
            _lib.check(_lib.load().alto_cast_f32_f64(tmp.data_ptr(), out.data_ptr(), tmp.numel(),
                                                     _lib.stream_ptr()), "alto_cast_f32_f64")
        return out
    a, _keep = _args(tensor, fdev, mode, out, tile, 1 if zero_out else 0)
    ms = (mode_stream(tensor, mode) if planned is True and PLAN_VARIANT == "pos"
          and _use_mode_stream(tensor, rank, fdev[0].element_size()) else None)
    if ms is not None:
        _set_stream(a, ms)
        tabs = []  # product tables: stream-ordered, released after the launch
        _set_pairs(a, tensor, fdev, mode, tabs)
    elif planned and tensor.nnz > 0 and rank in (16, 32) and 3 <= tensor.layout.order <= 5 \
            and max(tensor.layout.bits) <= 31:
        a.packed = packed_keys(tensor).data_ptr()
        if planned == "pos" or (planned is True and PLAN_VARIANT == "pos"):
            a.pos = subtile_order(tensor, mode).data_ptr()
        else:
            sp = stream_plan(tensor, mode, rank, fdev[0].element_size())
            a.plan = sp["plan"].data_ptr()
            for i, rws in enumerate(sp["cache_rows"]):
                a.cache_rows[i] = rws.data_ptr()
            a.cache_k = sp["k"]
            a.cache_modes = sp["modes"]
    if hot:
        _set_hot(a, tensor, mode, rank, out.dtype, ms)
    _lib.check(_lib.load().alto_mttkrp(ctypes.byref(a), _lib.stream_ptr()), "alto_mttkrp")
    return out


def row_index(tensor: AltoTensor, mode: int):
    """Per-mode (row_perm, row_ptr): elements sorted by (coordinate, position), cached."""
    torch = _torch()
    key = ("row_index", mode)
    hit = tensor._cache.get(key)
    if hit is not None:
        return hit
    lib = _lib.load()
    lay = tensor.layout
    m = tensor.nnz
    dim = lay.dims[mode]
    dev = tensor.keys.device
    perm = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    ptr = torch.empty(dim + 1, dtype=torch.int64, device=dev)
    ws_bytes = lib.alto_row_index_workspace_bytes(m, dim)
    ws = torch.empty(max(int(ws_bytes), 8), dtype=torch.uint8, device=dev)
    _lib.check(lib.alto_row_index(c_layout(lay), device_tables(lay).data_ptr(), tensor.keys.data_ptr(), m, mode,
                                  perm.data_ptr(), ptr.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_ptr()),
               "alto_row_index")
    tensor._cache[key] = (perm, ptr)
    return perm, ptr


# Rows longer than this make the exact-order engine's sequential per-row sums
# slow (a Zipf head row of 6.5M elements takes ~3 s); above it the
# deterministic fixed-point streaming path is used instead.
EXACT_MAX_RUN = int(__import__("os").environ.get("ALTO_EXACT_MAX_RUN", 65536))


def max_row_length(tensor: AltoTensor, mode: int) -> int:
    key = ("maxrun", mode)
    hit = tensor._cache.get(key)
    if hit is None:
        _perm, ptr = row_index(tensor, mode)
        hit = int((ptr[1:] - ptr[:-1]).max().item()) if ptr.numel() > 1 else 0
        tensor._cache[key] = hit
    return hit


def det_supported(tensor: AltoTensor, fdev: list) -> bool:
    torch = _torch()
    lay = tensor.layout
    rank = int(fdev[0].shape[1])
    return tensor.nnz > 0 and rank in (16, 32) and 3 <= lay.order <= 5 and max(lay.bits) <= 31


def mttkrp_det(tensor: AltoTensor, fdev: list, mode: int, out=None):
    """Deterministic streaming MTTKRP -> (I_mode, R) float64 device tensor.

    Same kernel as mttkrp_stream, but row partials are merged as int64 fixed
    point (scale = a power of two from the bound sum|v| * prod max|F|):
    integer addition is associative, so the result is bitwise identical for
    every run, tile order, worker or partition count."""
    torch = _torch()
    lib = _lib.load()
    dev = tensor.keys.device
    rank = int(fdev[0].shape[1])
    dim = tensor.layout.dims[mode]
    vals = tensor.vals
    if fdev[0].dtype != vals.dtype:
        # mixed precision: compute in float64 (upcasting float32 is exact)
        if vals.dtype == torch.float32:
            vals = tensor._cache.get("vals64")
            if vals is None:
                vals = tensor.vals.double()
                tensor._cache["vals64"] = vals
        else:
            fdev = [f.double() for f in fdev]
    ws = tensor._cache.get("det_ws")
    if ws is None:
        nb = int(lib.alto_cpd_workspace_bytes(1))
        ws = (torch.empty(nb, dtype=torch.uint8, device=dev), nb,
              torch.empty(_lib.ALTO_MAX_ORDER + 1, dtype=torch.float64, device=dev),
              torch.empty(1, dtype=torch.float64, device=dev))
        code = _lib.ALTO_F32 if tensor.vals.dtype == torch.float32 else _lib.ALTO_F64
        _lib.check(lib.alto_sumabs(tensor.vals.data_ptr(), code, tensor.nnz, ws[2].data_ptr(), ws[0].data_ptr(), nb,
                                   _lib.stream_ptr()), "alto_sumabs")
        tensor._cache["det_ws"] = ws
    buf, nb, terms, scale = ws
    k = 1
    for n, f in enumerate(fdev):
        if n == mode:
            continue
        code = _lib.ALTO_F32 if f.dtype == torch.float32 else _lib.ALTO_F64
        _lib.check(lib.alto_absmax(f.data_ptr(), code, f.numel(), terms[k:].data_ptr(), buf.data_ptr(), nb,
                                   _lib.stream_ptr()), "alto_absmax")
        k += 1
    _lib.check(lib.alto_fixed_scale(terms.data_ptr(), k, scale.data_ptr(), _lib.stream_ptr()), "alto_fixed_scale")
    fixed = torch.empty((dim, rank), dtype=torch.int64, device=dev)
    a, _keep = _args(tensor, fdev, mode, fixed, DEFAULT_TILE, 1, vals=vals)
    a.out_dtype = _lib.ALTO_I64
    a.fixed_scale = scale.data_ptr()
    ms = mode_stream(tensor, mode, vals) if _use_mode_stream(tensor, rank, fdev[0].element_size()) else None
    if ms is not None:
        _set_stream(a, ms)
    else:
        a.packed = packed_keys(tensor).data_ptr()
        a.pos = subtile_order(tensor, mode).data_ptr()
    _set_hot(a, tensor, mode, rank, torch.int64, ms)
    _lib.check(lib.alto_mttkrp(ctypes.byref(a), _lib.stream_ptr()), "alto_mttkrp(deterministic)")
    if out is None:
        out = torch.empty((dim, rank), dtype=torch.float64, device=dev)
    _lib.check(lib.alto_fixed_to_float(fixed.data_ptr(), scale.data_ptr(), out.data_ptr(), _dt_code(out),
                                       fixed.numel(), _lib.stream_ptr()), "alto_fixed_to_float")
    return out


def mttkrp_deterministic(tensor: AltoTensor, fdev: list, mode: int, part_offsets=None, out=None):
    """Deterministic MTTKRP: the exact-order engine (bitwise equal to the
    reference) when the longest row is short, else the fixed-point streaming
    kernel (bitwise reproducible, ~1e-13 relative to the exact sums)."""
    if tensor.nnz > 0 and det_supported(tensor, fdev) and max_row_length(tensor, mode) > EXACT_MAX_RUN:
        return mttkrp_det(tensor, fdev, mode, out=out)
    return mttkrp_exact(tensor, fdev, mode, part_offsets, out=out)


def mttkrp_exact(tensor: AltoTensor, fdev: list, mode: int, part_offsets=None, out=None):
    """Deterministic exact-order MTTKRP -> (I_mode, R) float64 device tensor."""
    torch = _torch()
    rank = int(fdev[0].shape[1])
    dim = tensor.layout.dims[mode]
    dev = tensor.keys.device
    if out is None:
        out = torch.empty((dim, rank), dtype=torch.float64, device=dev)
    if part_offsets is None:
        part_offsets = np.asarray([0, tensor.nnz], dtype=np.int64)
    offs = np.asarray(part_offsets, dtype=np.int64)
    key = ("part_off", offs.tobytes())
    d_off = tensor._cache.get(key)
    if d_off is None:
        d_off = torch.from_numpy(offs.copy()).to(dev)
        tensor._cache[key] = d_off
    perm, ptr = row_index(tensor, mode)
    a, _keep = _args(tensor, fdev, mode, out)
    _lib.check(_lib.load().alto_mttkrp_exact(ctypes.byref(a), perm.data_ptr(), ptr.data_ptr(), d_off.data_ptr(),
                                             len(offs) - 1, _lib.stream_ptr()), "alto_mttkrp_exact")
    return out


def _finish(out_dev, like_torch: bool):
    return out_dev if like_torch else out_dev.cpu().numpy()


def mttkrp_oracle(tensor: CooTensor, factors, mode: int):
    """COO MTTKRP (mttkrp.py:64-77) on the device, float64 atomics."""
    torch = _torch()
    rank = _check_factors(tensor.dims, factors, mode)
    dev = _lib.cuda_device()
    out = torch.empty((tensor.dims[mode], rank), dtype=torch.float64, device=dev)
    fdev = factors_to_device(factors, torch.float64, skip=mode)
    coords = torch.from_numpy(tensor.coords).to(dev)
    vals = torch.from_numpy(tensor.values).to(dev)
    arr = (ctypes.c_void_p * len(fdev))(*[f.data_ptr() for f in fdev])
    _lib.check(_lib.load().alto_mttkrp_coo(coords.data_ptr(), vals.data_ptr(), tensor.nnz, tensor.order, mode, rank,
                                           arr, out.data_ptr(), tensor.dims[mode], _lib.stream_ptr()),
               "alto_mttkrp_coo")
    return _finish(out, any(_is_torch(f) for f in factors))


def mttkrp_seq(tensor: AltoTensor, factors, mode: int):
    """Sequential-order MTTKRP (mttkrp.py:108-117): exact-order engine, one partition."""
    _check_factors(tensor.layout.dims, factors, mode)
    fdev = factors_to_device(factors, skip=mode)
    return _finish(mttkrp_deterministic(tensor, fdev, mode), any(_is_torch(f) for f in factors))


def _any_flag(tensor: AltoTensor, flag_bit: int) -> bool:
    """Whether any element carries `flag_bit` (the reference's `flags.any()`
    guard, mttkrp.py:192-200).  The answer is cached on the tensor (its keys
    are read-only; flagging returns a new tensor), so repeated calls do not
    re-read the keys or synchronize the host with the device."""
    if tensor.nnz == 0:
        return False
    key = ("anyflag", flag_bit)
    hit = tensor._cache.get(key)
    if hit is None:
        hit = bool(read_flags_device(tensor, flag_bit).any().item())
        tensor._cache[key] = hit
    return hit


def mttkrp_par(tensor: AltoTensor, parts: PartitionSet, plan: ConflictPlan, factors, mode: int,
               workers: int = 1):
    """Plan-driven MTTKRP (mttkrp.py:227-251).

    Buffered plans run the exact-order engine over the plan's partitions
    (bitwise deterministic, independent of `workers`); Atomic plans run the
    streaming kernel.  `workers` is validated but has no effect on device.
    """
    _check_factors(tensor.layout.dims, factors, mode)
    if workers < 1:
        raise ValueError("workers must be at least 1")
    if plan.mode != mode:
        raise ValueError(f"plan is for mode {plan.mode}, kernel asked for {mode}")
    if not np.array_equal(plan.offsets, parts.offsets):
        raise ValueError("plan and partition set do not match")
    fdev = factors_to_device(factors, skip=mode)  # the output mode's factor is never read
    like = any(_is_torch(f) for f in factors)
    if plan.strategy is Strategy.BUFFERED:
        return _finish(mttkrp_deterministic(tensor, fdev, mode, np.asarray(parts.offsets)), like)
    if plan.flag_bit is not None and plan.overlaps is not None and any(plan.overlaps) and tensor.nnz:
        if not _any_flag(tensor, plan.flag_bit):
            raise ValueError("plan expects boundary flags; apply_boundary_flags first")
    return _finish(mttkrp_stream(tensor, fdev, mode), like)


def mttkrp(tensor: AltoTensor, factors, mode: int, workers: int = 1, partitions: int | None = None,
           strategy: Strategy | None = None):
    """Partition, plan, flag if needed, and run (mttkrp.py:254-271)."""
    torch = _torch()
    rank = _check_factors(tensor.layout.dims, factors, mode)
    if tensor.nnz == 0:
        z = np.zeros((tensor.layout.dims[mode], rank), dtype=np.float64)
        return torch.from_numpy(z).to(_lib.cuda_device()) if any(_is_torch(f) for f in factors) else z
    count = min(partitions if partitions is not None else workers, tensor.nnz)
    parts = partition(tensor, max(count, 1))
    plan = plan_conflicts(tensor, parts, mode, force_strategy=strategy)
    if plan.strategy is Strategy.ATOMIC and plan.flag_bit is not None:
        tensor = apply_boundary_flags(tensor, plan)
    return mttkrp_par(tensor, parts, plan, factors, mode, workers)
