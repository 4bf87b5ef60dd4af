"""MTTKRP on the B200: drop-in for pkg/src/altotensor/mttkrp.py.

Engines (all device code in libalto_b200.so):
  * K8/K9 pull engine (`mttkrp_pull`, alto_mttkrp_pull, csrc/alto_pull.cuh)
    over the mode's row-major stream: slice interval buffers + a fixed-order
    float64 pull reduction — the reference's Buffered scheme
    (mttkrp.py:132-175), bitwise reproducible and independent of
    workers/partitions; with atomic=True its Atomic scheme (mttkrp.py:178-224:
    rows shared between slices merge with atomics, owned rows are stored).
    Buffered plans of large tensors and Atomic plans run here.
  * exact-order engine (`mttkrp_exact`, alto_mttkrp_exact) — per-row sums in
    element order, split at partition boundaries and merged in ascending
    partition order, in float64: exactly the arithmetic order of mttkrp_seq
    (mttkrp.py:108-117) and of the Buffered stage + pull (mttkrp.py:148-172),
    so results are bitwise equal to the reference on float64 inputs.  Used
    for Buffered plans of tensors up to EXACT_MAX_NNZ elements with rows of
    at most EXACT_MAX_RUN elements.
  * mode-stream kernel (`mttkrp_stream`, alto_mttkrp, csrc/alto_mstream.cuh)
    — the fastest float32 path (round-robin lane groups, RED merges,
    replicated hot rows); not bitwise reproducible (float atomics).  The
    bench's device-timed step and the `atomic` CP-ALS backend.
  * fixed-point streaming (`mttkrp_det`): int64 merges, deterministic; only a
    fallback for shapes the pull engine does not cover.  Its scale comes
    from a global bound, so rows of small magnitude keep fewer digits.
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
F32_ACCUMULATE = True
# Streaming-kernel switches (ALTO_STREAM_* in include/alto_b200.h; 0 = default).
STREAM_FLAGS = 0


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


# Pinned host factors are uploaded on a side stream.  By default the side
# stream first waits for the current stream, so work the caller queued
# before the call (e.g. a non_blocking device->host copy filling the pinned
# factor) completes before the upload reads it.  OVERLAP_UPLOADS = True drops
# that wait so an upload overlaps the previous call's kernels (bench.py's
# end-to-end leg opts in: its pinned inputs are written once, up front).
OVERLAP_UPLOADS = False


def factors_to_device(factors, dtype=None, skip: int | None = None) -> list:
    """Factors as contiguous device tensors (float64 unless dtype/torch input
    says otherwise).  `skip`: a host factor the MTTKRP of that mode never
    reads (the output mode's) is not copied; a 1-row placeholder of the same
    dtype and rank stands in for it.  Pinned host torch tensors are copied
    asynchronously on a side stream that the current stream then waits for
    (the side stream waits for the current stream first unless
    OVERLAP_UPLOADS is set; as with any non_blocking copy, a pinned input
    must not be modified until the stream is synchronized)."""
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
                if not OVERLAP_UPLOADS:
                    side.wait_stream(cur)  # pending writes to the pinned inputs land first
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
    return a, cl


# Hot-row plan: rows holding more than HOT_TAU elements appear in almost every
# tile; their tile partials go to replicated copies (a per-row number of
# them, alto_hot_copies) instead of contending on one L2 line (see
# alto_mttkrp_args in include/alto_b200.h).
HOT_TAU = 1024
HOT_MAX = 32768


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
        ptr = row_ptr(tensor, mode)
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


# Hot plan: at most HOT_BOUND merges per replicated copy of a hot row (bounds
# same-address contention and float32 rounding of the copies), at most
# 2^HOT_MAX_LG copies per row.
HOT_BOUND = 1024
HOT_MAX_LG = 10


def hot_plan_ms(tensor: AltoTensor, mode: int, rank: int, out_dtype, alto_order: bool = False):
    """Hot-row plan with per-row copy counts (alto_hot_copies), cached:
    (hot_code (I_mode,) int32, hot rows, count, hot_base (count+1,) int32, zeroed copies) or None.
    alto_order: for the kernels that walk the ALTO stream in 128-element
    sub-tiles (a row merges once per sub-tile it appears in), else for the
    mode stream."""
    torch = _torch()
    T = 128 if alto_order else ms_tile(tensor)
    order = 0 if alto_order else MS_ORDER
    key = ("hotms", mode, rank, out_dtype, T, order)
    if key in tensor._cache:
        return tensor._cache[key]
    hs = hot_slots(tensor, mode)
    plan = None
    if hs is not None:
        _slot, rows, n = hs
        dev = tensor.keys.device
        ptr = row_ptr(tensor, mode)
        code = torch.full((tensor.layout.dims[mode],), -1, dtype=torch.int32, device=dev)
        base = torch.empty(n + 1, dtype=torch.int32, device=dev)
        _lib.check(_lib.load().alto_hot_copies(ptr.data_ptr(), rows.data_ptr(), n, tensor.nnz, T, order, HOT_BOUND,
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
    # ALTO-order kernels: the same per-row copy counts, sized for one merge per
    # 128-element sub-tile a row appears in (bounded merges per float32 copy:
    # the uniform 64-copy plan left 3e-5 on cfg5's Zipf head at full size)
    hp = hot_plan_ms(tensor, mode, rank, out_dtype, alto_order=True)
    if hp is not None:
        code, rows, n, base, buf = hp
        a.hot_slot, a.hot_rows, a.n_hot, a.hot_copies, a.hot_buf, a.hot_base = (
            code.data_ptr(), rows.data_ptr(), n, 1, buf.data_ptr(), base.data_ptr())


# Per-mode stream tile length (elements); 0 disables the mode-stream kernel.
MS_TILE = 1024
# Mode-stream order: 1 (default) = the whole stream sorted by the mode's
# coordinate, ALTO order kept within a row (ALTO_MS_ROW_MAJOR); 0 = each tile
# (a contiguous ALTO key range) sorted by it.
MS_ORDER = 1
# Lane groups of a warp.  1 = round-robin positions s, s+8, ... of a tile
# (cooperative decode + shuffles); 0 = contiguous slices; 2 (default) = the
# blocked kernel (ALTO_MS_BLOCKED: same round-robin assignment, each group's
# elements of a warp step stored contiguously, every lane loads its group's
# keys/values itself with broadcast vector loads, no shuffles) for the shapes
# it wins on — rank 32 and orders 4-5: cfg3 2.64-2.77 -> 2.32-2.38 ms, cfg4
# 0.265 -> 0.239 ms per mode — and round robin for order 3 / rank 16, where it
# loses (cfg2 0.46 -> 0.50, cfg5 6.1 -> 6.6 ms; profiles/r02e_ab_blocked.jsonl);
# 3 = blocked wherever it exists.  Tile-ordered streams (MS_ORDER 0) use 1.
MS_RR = 2
# 128-bit layouts: store the mode stream with one key word per element (the
# input coordinates + the row increment within the lane group, ALTO_MS_DELTA)
# instead of two: 12 instead of 20 bytes per element on cfg3/cfg5.
MS_DELTA = 1
ALTO_MS_DELTA = 8
ALTO_MS_BLOCKED = 16


def ms_tile(tensor: AltoTensor) -> int:
    """Tile length of the tensor's mode streams: MS_TILE, halved (down to 128)
    for small tensors so that there are >= ~4 tiles per resident warp
    (148 SMs x 24 warps)."""
    t = MS_TILE
    while t > 128 and tensor.nnz < 148 * 24 * 4 * t:
        t //= 2
    return t


def ms_block(order: int, rank: int, vals_dtype_code: int, n_pairs: int):
    """(u, groups) of the blocked mode-stream kernel's warp step
    (alto_mstream_block), or None when no blocked kernel covers the shape."""
    u, g = ctypes.c_int32(0), ctypes.c_int32(0)
    rc = _lib.load().alto_mstream_block(order, rank, vals_dtype_code, n_pairs, ctypes.byref(u), ctypes.byref(g))
    if rc == _lib.ALTO_EUNSUPPORTED:
        return None
    _lib.check(rc, "alto_mstream_block")
    return int(u.value), int(g.value)


def _ms_group_mode(tensor: AltoTensor, vals, rank: int, n_pairs: int):
    """-> (rr, blk): the lane-group assignment the stream is built for.
    MS_RR = 2 picks the blocked kernel for the shapes it is the measured
    winner on (rank 32, orders 4-5; float32) and round robin elsewhere;
    MS_RR = 3 forces it wherever a blocked kernel exists (tests)."""
    torch = _torch()
    rr = MS_RR if MS_ORDER == 1 else min(MS_RR, 1)
    if rr == 2 and not (vals.dtype == torch.float32 and (rank == 32 or tensor.layout.order >= 4)):
        rr = 1
    rr = min(rr, 2)
    blk = ms_block(tensor.layout.order, rank, _dt_code(vals), n_pairs) if rr == 2 else None
    if rr == 2 and blk is None:
        rr = 1
    return rr, blk


def mode_stream_key(tensor: AltoTensor, mode: int, vals=None, rank: int = 16, n_pairs: int = 0):
    """Cache key of mode_stream (a blocked stream's storage order and delta
    encoding depend on the kernel's step shape)."""
    vals = tensor.vals if vals is None else vals
    rr, blk = _ms_group_mode(tensor, vals, rank, n_pairs)
    return ("mstream", mode, vals.dtype, ms_tile(tensor), MS_ORDER, rr, blk)


def mode_stream(tensor: AltoTensor, mode: int, vals=None, rank: int = 16, n_pairs: int = 0):
    """Per-mode stream of the MTTKRP (alto_mode_stream), cached per (mode,
    value dtype, lane-group assignment): the ALTO elements stably sorted by
    their `mode` coordinate (ALTO order kept within a row; tile by tile when
    MS_ORDER is 0), with hot-row flags.  `rank` / `n_pairs` select the blocked
    kernel's step shape.  -> (keys, values, tile, rr, base rows or None)."""
    torch = _torch()
    vals = tensor.vals if vals is None else vals
    T = ms_tile(tensor)
    rr, blk = _ms_group_mode(tensor, vals, rank, n_pairs)
    gflags = {0: 0, 1: 4}.get(rr, 0) if rr != 2 else (ALTO_MS_BLOCKED | (blk[0] << 8) | (blk[1] << 12))
    key = mode_stream_key(tensor, mode, vals, rank, n_pairs)
    hit = tensor._cache.get(key)
    if hit is None:
        lib = _lib.load()
        lay = tensor.layout
        m = tensor.nnz
        dev = tensor.keys.device
        hs = hot_slots(tensor, mode)
        hot = hs is not None and lay.total_bits < 64 * lay.n_words
        ntiles = (m + T - 1) // T
        wsb = int(lib.alto_mode_stream_workspace_bytes(m))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        svals = torch.empty(max(ntiles * T, 1), dtype=vals.dtype, device=dev)
        hit = None
        if MS_DELTA and lay.n_words == 2 and MS_ORDER == 1:
            # one key word per element: inputs + row increment (ALTO_MS_DELTA)
            skeys = torch.empty((max(ntiles * T, 1), 1), dtype=tensor.keys.dtype, device=dev)
            base = torch.empty(max(ntiles * 8, 1), dtype=torch.int32, device=dev)
            ovf = torch.empty(1, dtype=torch.int32, device=dev)
            rc = lib.alto_mode_stream(c_layout(lay), packed_keys(tensor).data_ptr(), vals.data_ptr(), _dt_code(vals),
                                      m, mode, T, MS_ORDER | gflags | ALTO_MS_DELTA,
                                      hs[0].data_ptr() if hot else None, skeys.data_ptr(), svals.data_ptr(),
                                      base.data_ptr(), ovf.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr())
            if rc != _lib.ALTO_EUNSUPPORTED:
                _lib.check(rc, "alto_mode_stream(delta)")
                if int(ovf.item()) == 0:
                    hit = (skeys, svals, T, rr, base)
            del skeys, base
        if hit is None:
            skeys = torch.empty((max(ntiles * T, 1), lay.n_words), dtype=tensor.keys.dtype, device=dev)
            rc = lib.alto_mode_stream(c_layout(lay), packed_keys(tensor).data_ptr(), vals.data_ptr(), _dt_code(vals),
                                      m, mode, T, MS_ORDER | gflags, hs[0].data_ptr() if hot else None,
                                      skeys.data_ptr(), svals.data_ptr(), None, None, ws.data_ptr(), wsb,
                                      _lib.stream_ptr())
            if rc == _lib.ALTO_EUNSUPPORTED:
                hit = False  # field layout does not fit the key width: planned kernel instead
            else:
                _lib.check(rc, "alto_mode_stream")
                hit = (skeys, svals, T, rr, None)
        del ws
        tensor._cache[key] = hit
    return hit or None


# L2 residency budget (MB) for the gathered factors of the mode-stream kernel
# on tensors whose factors exceed the L2 (alto_mttkrp_args.l2_hot_bytes): the
# budget is split over the input modes (small factors whole, the rest evenly);
# rows must be numbered by popularity for the leading bytes to be the hot ones
# (the synthetic configs are).  0 = default L2 policy.
MS_L2_HOT_MB = 0


def l2_hot_bytes(dims, mode: int, rank: int, fbytes: int = 4, budget_mb: float | None = None):
    """Per-mode leading bytes gathered with the L2 evict_last policy."""
    budget = int((MS_L2_HOT_MB if budget_mb is None else budget_mb) * (1 << 20))
    out = [0] * len(dims)
    ins = sorted((n for n in range(len(dims)) if n != mode), key=lambda n: dims[n])
    sizes = {n: dims[n] * rank * fbytes for n in ins}
    if budget <= 0 or sum(sizes.values()) <= budget:
        return out  # everything fits anyway: leave the default policy
    left = budget
    for i, n in enumerate(ins):
        share = left // (len(ins) - i)
        out[n] = int(min(sizes[n], share, (1 << 32) - 1))
        left -= out[n]
    return out


def _set_stream(a, ms) -> None:
    sk, sv, st, rr, base = ms
    a.mkeys, a.mvals, a.mtile, a.mrr = sk.data_ptr(), sv.data_ptr(), st, int(rr)
    a.mbase = None if base is None else base.data_ptr()


# Ranks served by the mode-stream kernel (others: the planned ALTO-order
# kernel).  Rank 32 joined in round 2: with one-word delta keys cfg3 modes
# 0-1 run 2.74 / 2.64 ms vs 2.90 / 2.78 on the planned kernel.
MS_RANKS = (16, 32)


# Paired input modes (orders 4-5, float32, rank 16): two input modes whose
# row-wise product table (I_a * I_b rows) stays within MS_PAIR_BYTES are
# gathered as one row, so one gather replaces two (0 disables pairing).
MS_PAIR_BYTES = 64 << 20


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
    npairs = (len(ms_pairs(tensor.layout.dims, mode, rank, 4))
              if tensor.vals.dtype == torch.float32 and fdev[0].dtype == torch.float32 else 0)
    ms = (mode_stream(tensor, mode, rank=rank, n_pairs=npairs)
          if planned is True and _use_mode_stream(tensor, rank, fdev[0].element_size()) else None)
    if ms is not None:
        _set_stream(a, ms)
        tabs = []  # product tables: stream-ordered, released after the launch
        _set_pairs(a, tensor, fdev, mode, tabs)
        if MS_L2_HOT_MB and fdev[0].dtype == torch.float32 and out.dtype == torch.float32:
            for n, b in enumerate(l2_hot_bytes(tensor.layout.dims, mode, rank, 4)):
                a.l2_hot_bytes[n] = b
    elif planned and tensor.nnz > 0 and rank in (16, 32) and 3 <= tensor.layout.order <= 5 \
            and max(tensor.layout.bits) <= 31:
        # the single ALTO-order copy: packed keys + per-mode sub-tile order
        a.packed = packed_keys(tensor).data_ptr()
        a.pos = subtile_order(tensor, mode).data_ptr()
        tabs = []  # product tables of paired input modes (orders 4-5, rank 16, float32)
        if out.dtype != torch.int64:
            _set_pairs(a, tensor, fdev, mode, tabs)
    if hot:
        _set_hot(a, tensor, mode, rank, out.dtype, ms)
    _lib.check(_lib.load().alto_mttkrp(ctypes.byref(a), _lib.stream_ptr()), "alto_mttkrp")
    return out


# ---- K8/K9: slice interval buffers + deterministic pull (alto_pull.cuh) ----
# Records per level-1 pull chunk (kPullChunk in csrc/alto_pull.cuh).
PULL_CHUNK = 64
ALTO_MS_ROW_MAJOR = 1
# Pull-stream tile for large tensors (slices of PULL_TILE / 8 stream
# positions; >= 8 slices per resident lane group), else the mode-stream tile.
# Measured on cfg5 (ms per mode): 1024 -> 6.82 / 6.70 / 7.25, 2048 -> 6.57 /
# 6.47 / 6.96, 4096 -> 6.43 / 6.32 / 6.83, 8192 -> 6.45 / 6.39 / 6.87
# (fewer boundary records, longer runs); shorter slices are slower.
PULL_TILE = 4096

def pull_stream(tensor: AltoTensor, mode: int):
    """The mode's row-major stream with contiguous slices (alto_mode_stream,
    ALTO_MS_ROW_MAJOR): the ALTO elements stably sorted by the output
    coordinate, ALTO order kept inside a row, cached per (mode, tile) like the
    reference's per-mode plans (_make_backend, cpd.py:149-181).  128-bit
    layouts use one-word delta keys (ALTO_MS_DELTA) when the increments fit.
    -> (keys, values, tile, base rows or None) or None when the field layout
    does not fit."""
    torch = _torch()
    T = PULL_TILE if tensor.nnz >= 148 * 24 * 8 * PULL_TILE else ms_tile(tensor)
    key = ("pstream", mode, T)
    hit = tensor._cache.get(key)
    if hit is None:
        lib = _lib.load()
        lay = tensor.layout
        m = tensor.nnz
        dev = tensor.keys.device
        vals = tensor.vals
        ntiles = (m + T - 1) // T
        svals = torch.empty(max(ntiles * T, 1), dtype=vals.dtype, device=dev)
        wsb = int(lib.alto_mode_stream_workspace_bytes(m))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        if MS_DELTA and lay.n_words == 2 and vals.dtype == torch.float32:
            skeys = torch.empty((max(ntiles * T, 1), 1), dtype=tensor.keys.dtype, device=dev)
            base = torch.empty(max(ntiles * 8, 1), dtype=torch.int32, device=dev)
            ovf = torch.empty(1, dtype=torch.int32, device=dev)
            rc = lib.alto_mode_stream(c_layout(lay), packed_keys(tensor).data_ptr(), vals.data_ptr(), _dt_code(vals),
                                      m, mode, T, ALTO_MS_ROW_MAJOR | ALTO_MS_DELTA, None, skeys.data_ptr(),
                                      svals.data_ptr(), base.data_ptr(), ovf.data_ptr(), ws.data_ptr(), wsb,
                                      _lib.stream_ptr())
            if rc != _lib.ALTO_EUNSUPPORTED:
                _lib.check(rc, "alto_mode_stream(delta)")
                if int(ovf.item()) == 0:
                    hit = (skeys, svals, T, base)
        if hit is None:
            skeys = torch.empty((max(ntiles * T, 1), lay.n_words), dtype=tensor.keys.dtype, device=dev)
            rc = lib.alto_mode_stream(c_layout(lay), packed_keys(tensor).data_ptr(), vals.data_ptr(), _dt_code(vals),
                                      m, mode, T, ALTO_MS_ROW_MAJOR, None, skeys.data_ptr(), svals.data_ptr(),
                                      None, None, ws.data_ptr(), wsb, _lib.stream_ptr())
            if rc == _lib.ALTO_EUNSUPPORTED:
                hit = False
            else:
                _lib.check(rc, "alto_mode_stream")
                hit = (skeys, svals, T, None)
        del ws
        tensor._cache[key] = hit
    return hit or None


def pull_plan(tensor: AltoTensor, mode: int):
    """Shared-row plan of the pull engine for one mode, cached.

    A slice (T/8 consecutive positions of the row-major stream) owns every row
    strictly inside its output interval; its first / last row is shared when
    the neighbouring slice ends / starts with the same row (the rows
    apply_boundary_flags would flag, format.py:257-285).  Each shared run gets
    a record slot; a shared row's records are consecutive slots (element
    order), summed by the pull in chunks of PULL_CHUNK records and then over
    chunks.  Built on the device from the slices' first/last rows
    (alto_pull_slice_rows)."""
    torch = _torch()
    ps = pull_stream(tensor, mode)
    T = ps[2]
    key = ("pplan", mode, T)
    hit = tensor._cache.get(key)
    if hit is not None:
        return hit
    m = tensor.nnz
    dev = tensor.keys.device
    ch = T // 8
    ns = (m + ch - 1) // ch
    fl = torch.empty((max(ns, 1), 2), dtype=torch.int32, device=dev)
    _lib.check(_lib.load().alto_pull_slice_rows(c_layout(tensor.layout), ps[0].data_ptr(), m, mode, T,
                                                None if ps[3] is None else ps[3].data_ptr(), fl.data_ptr(),
                                                _lib.stream_ptr()), "alto_pull_slice_rows")
    first, last = fl[:ns, 0].long(), fl[:ns, 1].long()
    sf = torch.zeros(ns, dtype=torch.bool, device=dev)
    sl = torch.zeros(ns, dtype=torch.bool, device=dev)
    if ns > 1:
        sf[1:] = first[1:] == last[:-1]
        sl[:-1] = last[:-1] == first[1:]
    single = first == last
    cnt = torch.where(single, (sf | sl).long(), sf.long() + sl.long())
    start = torch.cumsum(cnt, 0) - cnt
    slot_x = torch.where(sf, start, torch.full_like(start, -1))
    slot_y = torch.where(sl, torch.where(single, start, start + sf.long()), torch.full_like(start, -1))
    slice_rec = torch.stack([slot_x, slot_y], 1).to(torch.int32).contiguous()
    n_rec = int(cnt.sum().item()) if ns else 0
    rec_row = torch.empty(max(n_rec, 1), dtype=torch.long, device=dev)
    rec_row[slot_x[sf]] = first[sf]
    rec_row[slot_y[sl]] = last[sl]
    rec_row = rec_row[:n_rec]
    if n_rec:
        change = torch.ones(n_rec, dtype=torch.bool, device=dev)
        change[1:] = rec_row[1:] != rec_row[:-1]
        seg_start = torch.nonzero(change).flatten()
        seg_row = rec_row[seg_start].to(torch.int32).contiguous()
        seg_off = torch.cat([seg_start, torch.tensor([n_rec], device=dev)])
        counts = seg_off[1:] - seg_off[:-1]
        nch = (counts + PULL_CHUNK - 1) // PULL_CHUNK
        seg_chunk_off = torch.cat([torch.zeros(1, dtype=torch.long, device=dev), torch.cumsum(nch, 0)])
        n_chunks = int(seg_chunk_off[-1].item())
        chunk_seg = torch.repeat_interleave(torch.arange(seg_row.numel(), device=dev), nch)
        j = torch.arange(n_chunks, device=dev) - seg_chunk_off[chunk_seg]
        chunk_off = torch.cat([seg_off[chunk_seg] + j * PULL_CHUNK, torch.tensor([n_rec], device=dev)]).contiguous()
        mseg = torch.nonzero(nch > 1).flatten().to(torch.int32).contiguous()
        chunk_seg = chunk_seg.to(torch.int32).contiguous()
    else:
        seg_row = torch.zeros(1, dtype=torch.int32, device=dev)
        seg_chunk_off = torch.zeros(1, dtype=torch.long, device=dev)
        chunk_off = torch.zeros(1, dtype=torch.long, device=dev)
        chunk_seg = torch.zeros(1, dtype=torch.int32, device=dev)
        mseg = torch.zeros(0, dtype=torch.int32, device=dev)
        n_chunks = 0
    hit = {"slice_rows": fl, "slice_rec": slice_rec, "n_rec": n_rec, "seg_row": seg_row, "n_seg": int(seg_row.numel()) if n_rec else 0,
           "chunk_off": chunk_off, "chunk_seg": chunk_seg, "seg_chunk_off": seg_chunk_off, "n_chunks": n_chunks,
           "mseg": mseg, "n_mseg": int(mseg.numel())}
    tensor._cache[key] = hit
    return hit


def pull_supported(tensor: AltoTensor, rank: int, fbytes: int, out_bytes: int = 8, atomic: bool = False) -> bool:
    """Shapes the pull engine covers (else the caller uses another engine)."""
    lay = tensor.layout
    if not (tensor.nnz > 0 and 3 <= lay.order <= 5 and max(lay.bits) <= 31 and tensor.nnz < (1 << 32) - 1):
        return False
    f32_only = fbytes == 4 and out_bytes == 4 and not atomic and tensor.vals.element_size() == 4
    return rank in (16, 32) or (rank in (8, 64) and f32_only)


def mttkrp_pull(tensor: AltoTensor, fdev: list, mode: int, out=None, out_dtype=None, atomic: bool = False):
    """K8/K9 MTTKRP -> (I_mode, R) device tensor (float64 unless out/out_dtype
    says float32; float32 needs float32 values and factors).

    atomic=False (Buffered): owned rows stored, shared rows pulled in a
    fixed order -> bitwise reproducible.  atomic=True: shared rows merged
    with RED (the Atomic scheme).  float32 values with float64 factors are
    computed in float64 (the reference's arithmetic on upcast inputs).
    Returns None when the shape is not covered (the caller falls back)."""
    torch = _torch()
    rank = int(fdev[0].shape[1])
    dim = tensor.layout.dims[mode]
    vals = tensor.vals
    if vals.dtype == torch.float64 and fdev[0].dtype == torch.float32:
        fdev = [f.double() for f in fdev]  # exact upcast
    fb = fdev[0].element_size()
    if out is None:
        out = torch.empty((dim, rank), dtype=out_dtype or torch.float64, device=tensor.keys.device)
    if out.dtype == torch.float32 and (fb != 4 or vals.dtype != torch.float32):
        return None
    if not pull_supported(tensor, rank, fb, out.element_size(), atomic):
        return None
    ps = pull_stream(tensor, mode)
    if ps is None:
        return None
    plan = pull_plan(tensor, mode)
    lay = tensor.layout
    a = _lib.CPullArgs()
    cl = c_layout(lay)
    a.lay = ctypes.pointer(cl)
    a.mkeys, a.mvals, a.value_dtype, a.tile = ps[0].data_ptr(), ps[1].data_ptr(), _dt_code(vals), ps[2]
    a.m, a.mode, a.rank = tensor.nnz, mode, rank
    fdt = {_dt_code(f) for f in fdev}
    if len(fdt) != 1:
        raise ValueError("factor matrices must share one dtype")
    a.factor_dtype = fdt.pop()
    a.out_dtype = _dt_code(out)
    a.atomic = 1 if atomic else 0
    for n, f in enumerate(fdev):
        a.factors[n] = f.data_ptr()
    a.out = out.data_ptr()
    a.slice_rec = plan["slice_rec"].data_ptr()
    a.slice_rows = plan["slice_rows"].data_ptr()
    a.mbase = None if ps[3] is None else ps[3].data_ptr()
    tabs = []  # product tables of paired input modes: stream-ordered, released after the launch
    if fb == 4 and vals.dtype == torch.float32:
        _set_pairs(a, tensor, fdev, mode, tabs)
    rec = part = None
    if not atomic and plan["n_rec"]:
        rec = torch.empty((plan["n_rec"], rank), dtype=fdev[0].dtype, device=out.device)
        part = torch.empty((max(plan["n_chunks"], 1), rank), dtype=torch.float64, device=out.device)
    a.rec = None if rec is None else rec.data_ptr()
    a.part = None if part is None else part.data_ptr()
    a.n_seg, a.seg_row = plan["n_seg"], plan["seg_row"].data_ptr()
    a.n_chunks = plan["n_chunks"] if not atomic else 0
    a.chunk_off, a.chunk_seg = plan["chunk_off"].data_ptr(), plan["chunk_seg"].data_ptr()
    a.seg_chunk_off = plan["seg_chunk_off"].data_ptr()
    a.n_mseg, a.mseg = plan["n_mseg"], plan["mseg"].data_ptr() if plan["n_mseg"] else None
    rc = _lib.load().alto_mttkrp_pull(ctypes.byref(a), _lib.stream_ptr())
    if rc == _lib.ALTO_EUNSUPPORTED:
        return None
    _lib.check(rc, "alto_mttkrp_pull")
    return out


def row_ptr(tensor: AltoTensor, mode: int):
    """Per-mode row offsets (I_mode + 1,) int64 — the rows' element counts, which is all the
    hot-row plans need: the row index's if it is cached, else the prefix sum of
    alto_row_counts (a histogram: no sort, no 4-byte-per-element permutation kept)."""
    torch = _torch()
    hit = tensor._cache.get(("row_index", mode))
    if hit is not None:
        return hit[1]
    key = ("row_ptr", mode)
    ptr = tensor._cache.get(key)
    if ptr is None:
        lib = _lib.load()
        lay = tensor.layout
        m = tensor.nnz
        dim = lay.dims[mode]
        dev = tensor.keys.device
        counts = torch.zeros(max(dim, 1), dtype=torch.int32, device=dev)
        _lib.check(lib.alto_row_counts(c_layout(lay), device_tables(lay).data_ptr(), tensor.keys.data_ptr(), m, mode,
                                       counts.data_ptr(), _lib.stream_ptr()), "alto_row_counts")
        ptr = torch.zeros(dim + 1, dtype=torch.int64, device=dev)
        # counts are uint32 in an int32 tensor (a row holds fewer than 2^32 elements): widen without sign
        torch.cumsum(counts[:dim].to(torch.int64) & 0xFFFFFFFF, 0, out=ptr[1:])
        tensor._cache[key] = ptr
    return ptr


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
EXACT_MAX_RUN = 65536


def max_row_length(tensor: AltoTensor, mode: int) -> int:
    key = ("maxrun", mode)
    hit = tensor._cache.get(key)
    if hit is None:
        ptr = row_ptr(tensor, mode)
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
    if not bool(torch.isfinite(terms[:k]).all().item()):
        # a NaN/Inf value or factor has no fixed-point bound: the exact-order
        # engine propagates it like the reference does
        return mttkrp_exact(tensor, fdev, mode, out=out)
    fixed = torch.empty((dim, rank), dtype=torch.int64, device=dev)
    a, _keep = _args(tensor, fdev, mode, fixed, DEFAULT_TILE, 1, vals=vals)
    a.out_dtype = _lib.ALTO_I64
    a.fixed_scale = scale.data_ptr()
    ms = (mode_stream(tensor, mode, vals, rank=rank)
          if _use_mode_stream(tensor, rank, fdev[0].element_size()) else None)
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


# Buffered plans up to this many elements (with rows no longer than
# EXACT_MAX_RUN) run the exact-order engine, bitwise equal to the reference;
# larger tensors run the K8/K9 pull engine (bitwise reproducible, ~1e-16
# relative to the exact sums in float64).
EXACT_MAX_NNZ = 4_000_000


def mttkrp_deterministic(tensor: AltoTensor, fdev: list, mode: int, part_offsets=None, out=None, out_dtype=None):
    """Deterministic MTTKRP (the Buffered scheme, mttkrp.py:132-175).

    * small tensors with short rows: the exact-order engine (bitwise equal
      to the reference's Buffered / seq results on float64 data);
    * otherwise the K8/K9 pull engine (slice interval buffers + fixed-order
      float64 pull: bitwise reproducible, independent of workers/partitions);
    * shapes the pull engine does not cover: the fixed-point streaming kernel
      for long rows, else the exact-order engine."""
    big = tensor.nnz > EXACT_MAX_NNZ
    if tensor.nnz > 0 and (big or max_row_length(tensor, mode) > EXACT_MAX_RUN):
        r = mttkrp_pull(tensor, fdev, mode, out=out, out_dtype=out_dtype)
        if r is not None:
            return r
        if det_supported(tensor, fdev) and max_row_length(tensor, mode) > EXACT_MAX_RUN:
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
    """COO MTTKRP (mttkrp.py:64-77) on the device in the reference's order:
    each output row sums its elements in input order (np.add.at), products in
    ascending mode order, float64 without contraction — bitwise equal to the
    reference (alto_mttkrp_coo_ordered)."""
    torch = _torch()
    rank = _check_factors(tensor.dims, factors, mode)
    dev = _lib.cuda_device()
    lib = _lib.load()
    dim = tensor.dims[mode]
    out = torch.empty((dim, rank), dtype=torch.float64, device=dev)
    fdev = factors_to_device(factors, torch.float64, skip=mode)
    coords = torch.from_numpy(np.ascontiguousarray(tensor.coords, dtype=np.int64)).to(dev)
    vals = torch.from_numpy(np.ascontiguousarray(tensor.values, dtype=np.float64)).to(dev)
    arr = (ctypes.c_void_p * len(fdev))(*[f.data_ptr() for f in fdev])
    wsb = int(lib.alto_mttkrp_coo_workspace_bytes(tensor.nnz, dim))
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev)
    _lib.check(lib.alto_mttkrp_coo_ordered(coords.data_ptr(), vals.data_ptr(), tensor.nnz, tensor.order, mode, rank,
                                           arr, out.data_ptr(), dim, ws.data_ptr(), wsb, _lib.stream_ptr()),
               "alto_mttkrp_coo_ordered")
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

    Buffered plans run the deterministic engines (exact-order engine over the
    plan's partitions for small tensors, else the K8/K9 pull engine; bitwise
    reproducible, independent of `workers`); Atomic plans run the pull
    engine's atomic scheme.  `workers` is validated but has no effect on
    device.
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
    # Atomic scheme: rows shared between slices merge with atomics, owned
    # rows are stored directly (the pull engine's boundary flags); the
    # streaming kernel for shapes it does not cover
    out = mttkrp_pull(tensor, fdev, mode, atomic=True)
    return _finish(out if out is not None else mttkrp_stream(tensor, fdev, mode), like)


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
