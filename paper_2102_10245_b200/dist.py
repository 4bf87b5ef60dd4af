"""Key-range-sharded MTTKRP / CP-ALS across GPUs.

The reference has no distributed path (threads only, mttkrp.py:120-129; the
paper lists distributed memory as future work).  Here each rank
(one process per GPU, torch.distributed over NCCL) holds one contiguous
key range of the sorted ALTO stream — exactly an ALTO partition
(format.py:127-154) — and full-size factor matrices.

Shards (build_shard): every rank linearizes the coordinates it was handed
(K1), picks the cut keys from a strided sample so that the shards balance a
cost model — elements x (key + value bytes) plus, per mode, rows touched x
R x factor bytes (each sampled element carries 1/count of its row, so a
range's weight counts the rows it touches; Zipf tails make equal-nnz shards
unequal in gather cost) — and then sorts only the elements of its own key
range (K2).  The API-level `partition` stays equal-nnz.

Per mode n:
  1. local MTTKRP over the shard (rows touched only by this shard are final);
  2. owner-directed shared-row exchange (exchange_shared): every row touched
     by >= 2 shards has one owner (its lowest-rank toucher); the other
     touchers send their partial rows to the owner in one grouped
     send/recv (NCCL group: ncclSend/ncclRecv), the owner adds them in rank
     order (deterministic) and sends the reduced rows back to exactly the
     ranks that touch them — each rank moves only the shared rows it
     touches, never a global all-reduce over I_n or over all shared rows;
  3. every rank solves the rows it touches (X V = M); shared rows are
     solved redundantly by each toucher, so no factor rows are sent back;
  4. column norms, the Gram of the new factor and the fit inner product are
     reduced over *owned* rows only — R, R x R and 1 values per mode cross
     the interconnect.

All compute goes through an `ops` object: `DeviceOps` binds the B200 C ABI;
tests inject CPU ops (gloo backend) to exercise the exchange logic.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib


def _torch():
    import torch

    return torch


def _p2p(sends, recvs, group=None):
    """One grouped batch of point-to-point transfers (NCCL: ncclGroupStart /
    ncclSend x k / ncclRecv x k / ncclGroupEnd).  gloo only moves host
    tensors, so device buffers are staged through the host there."""
    torch = _torch()
    import torch.distributed as dist

    if not sends and not recvs:
        return
    stage = dist.get_backend(group) == "gloo"
    ops, post = [], []
    for t, peer in sends:
        ops.append(dist.P2POp(dist.isend, t.cpu() if (stage and t.is_cuda) else t, peer, group))
    for t, peer in recvs:
        if stage and t.is_cuda:
            h = torch.empty(t.shape, dtype=t.dtype)
            ops.append(dist.P2POp(dist.irecv, h, peer, group))
            post.append((t, h))
        else:
            ops.append(dist.P2POp(dist.irecv, t, peer, group))
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    for t, h in post:
        t.copy_(h)


class ShardRows:
    """Exchange plan of one mode: shared rows, owners, this rank's owned-row
    mask, and the owner-directed send/receive row lists."""

    def __init__(self, touched, group=None):
        torch = _torch()
        import torch.distributed as dist

        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        cnt = touched.to(torch.int32)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
        first = torch.where(touched, torch.full_like(cnt, rank), torch.full_like(cnt, world))
        dist.all_reduce(first, op=dist.ReduceOp.MIN, group=group)
        shared = cnt >= 2
        self.shared_rows = torch.nonzero(shared).flatten().to(torch.int64)
        self.owned = touched & ((cnt == 1) | (first == rank))
        self.mask = self.owned.to(torch.uint8)
        self.touched = touched
        self.group = group
        self.rank, self.world = rank, world
        # rows this rank sends to each owner (shared rows it touches but does not own)
        mine = touched & shared & (first != rank)
        rows = torch.nonzero(mine).flatten().to(torch.int64)
        owner = first[rows].to(torch.int64)
        self.send = {}
        for o in range(world):
            r = rows[owner == o]
            if r.numel():
                self.send[o] = r.contiguous()
        # tell every owner how many rows (and which) each rank will send it
        counts = torch.zeros(world, dtype=torch.int64, device=touched.device)
        for o, r in self.send.items():
            counts[o] = r.numel()
        allc = [torch.zeros_like(counts) for _ in range(world)]
        dist.all_gather(allc, counts, group=group)
        self.recv = {}
        recvs = []
        for r_ in range(world):
            n = int(allc[r_][rank].item())
            if r_ != rank and n:
                buf = torch.empty(n, dtype=torch.int64, device=touched.device)
                self.recv[r_] = buf
                recvs.append((buf, r_))
        _p2p([(r, o) for o, r in self.send.items()], recvs, group)

    @property
    def n_shared(self) -> int:
        return int(self.shared_rows.numel())

    def bytes_per_exchange(self, rank_r: int, elem_bytes: int) -> int:
        """Bytes this rank sends + receives in one exchange (both legs)."""
        rows = sum(int(r.numel()) for r in self.send.values()) + sum(int(r.numel()) for r in self.recv.values())
        return 2 * rows * rank_r * elem_bytes


def exchange_shared(out, plan: ShardRows, ops) -> None:
    """Owner-directed shared-row reduction of `out` (in place): non-owners send
    their partial rows to the owners, owners add them in rank order and send
    the reduced rows back to exactly the ranks that touch them."""
    torch = _torch()
    if not plan.send and not plan.recv:
        return
    R = out.shape[1]
    sends = [(ops.pack(out, rows), o) for o, rows in plan.send.items()]
    rbufs = {r: torch.empty((rows.numel(), R), dtype=out.dtype, device=out.device) for r, rows in plan.recv.items()}
    _p2p(sends, [(b, r) for r, b in rbufs.items()], plan.group)
    for r in sorted(rbufs):
        ops.add_rows(out, plan.recv[r], rbufs[r])
    back = [(ops.pack(out, rows), r) for r, rows in plan.recv.items()]
    bbufs = {o: torch.empty((rows.numel(), R), dtype=out.dtype, device=out.device) for o, rows in plan.send.items()}
    _p2p(back, [(b, o) for o, b in bbufs.items()], plan.group)
    for o, b in bbufs.items():
        ops.unpack(out, plan.send[o], b)


def build_shard(layout, coords, vals, rank: int, world: int, rank_r: int, sample: int = 1 << 22):
    """This rank's key-range shard, cut by a cost model and built from its
    own key range only (K1 on the given coordinates, K2 on the shard).

    Cost of a key range = elements x (K + V) + sum_n rows_touched_n x R x S,
    estimated on a strided sample whose elements weigh 1/count of their row
    (full per-mode row counts).  Returns (AltoTensor, info)."""
    torch = _torch()
    from .format import AltoTensor
    from .layout import linearize_device

    m = int(coords.shape[0])
    keys, bad = linearize_device(layout, coords)
    nw = layout.n_words
    kv = 8 * nw + vals.element_size()
    rs = rank_r * vals.element_size()
    step = max(1, m // sample)
    idx = torch.arange(0, m, step, device=coords.device)
    w = torch.full((idx.numel(),), float(kv) * step, dtype=torch.float64, device=coords.device)
    for n, d in enumerate(layout.dims):
        cnt = torch.bincount(coords[:, n], minlength=int(d)).to(torch.float64)
        w += rs * step / cnt[coords[idx, n]]
    sk = keys[idx]
    flip = torch.tensor(-(1 << 63), dtype=torch.int64, device=keys.device)  # unsigned order via signed compare
    if nw == 1:
        order = torch.argsort(sk[:, 0] ^ flip, stable=True)
    else:
        order = torch.argsort(sk[:, 0] ^ flip, stable=True)
        order = order[torch.argsort((sk[order, 1] ^ flip), stable=True)]
    cw = torch.cumsum(w[order], 0)
    total = float(cw[-1].item())
    pos = [int(torch.searchsorted(cw, torch.tensor(total * g / world, dtype=torch.float64,
                                                    device=cw.device)).item()) for g in range(1, world)]
    cuts = [sk[order[min(p, order.numel() - 1)]] for p in pos]  # first key of shard g (g >= 1)

    def ge(key_row):  # keys >= key_row (unsigned lexicographic, MS word last)
        if nw == 1:
            return (keys[:, 0] ^ flip) >= (key_row[0] ^ flip)
        hi, lo = keys[:, 1] ^ flip, keys[:, 0] ^ flip
        khi, klo = key_row[1] ^ flip, key_row[0] ^ flip
        return (hi > khi) | ((hi == khi) & (lo >= klo))

    sel = torch.ones(m, dtype=torch.bool, device=keys.device)
    if rank > 0:
        sel &= ge(cuts[rank - 1])
    if rank < world - 1:
        sel &= ~ge(cuts[rank])
    skeys = keys[sel].contiguous()
    svals = vals[sel].contiguous()
    del keys
    lib = _lib.load()
    ms = int(skeys.shape[0])
    ws_bytes = lib.alto_sort_workspace_bytes(ms, nw, svals.element_size())
    wsb = torch.empty(max(int(ws_bytes), 8), dtype=torch.uint8, device=skeys.device)
    _lib.check(lib.alto_sort_pairs(skeys.data_ptr(), svals.data_ptr(), ms, nw, svals.element_size(),
                                   layout.total_bits, wsb.data_ptr(), ws_bytes, _lib.stream_ptr()), "alto_sort_pairs")
    first = torch.empty(1, dtype=torch.int64, device=skeys.device)
    _lib.check(lib.alto_find_duplicate(skeys.data_ptr(), ms, nw, first.data_ptr(), _lib.stream_ptr()),
               "alto_find_duplicate")
    flags = torch.stack([bad[0], first[0]]).cpu()
    if int(flags[0]) >= 0:
        raise ValueError("coordinates out of range for layout dims")
    if int(flags[1]) >= 0:
        raise ValueError("duplicate coordinates; coalesce the tensor first")
    est = [float(cw[p - 1].item()) if p > 0 else 0.0 for p in pos]
    bounds = [0.0] + est + [total]
    info = {"nnz": ms, "cut": "cost-balanced key ranges (elements x (K+V) + touched rows x R x S)",
            "est_cost_share": [(bounds[g + 1] - bounds[g]) / total for g in range(world)]}
    return AltoTensor(layout, skeys, svals), info


class DeviceOps:
    """B200 implementations of the per-shard steps (libalto_b200.so)."""

    def __init__(self, shard, rank: int):
        from .cpd import _Workspace

        self.shard = shard
        self.rank = rank
        self.dev = shard.keys.device
        self.ws = _Workspace(rank, self.dev)
        self.lib = _lib.load()

    def touched_rows(self, mode: int):
        from .mttkrp import row_ptr

        ptr = row_ptr(self.shard, mode)
        return (ptr[1:] - ptr[:-1]) > 0

    def mttkrp(self, factors, mode: int):
        from .mttkrp import mttkrp_stream

        return mttkrp_stream(self.shard, factors, mode)

    def _dt(self, t):
        torch = _torch()
        return _lib.ALTO_F32 if t.dtype == torch.float32 else _lib.ALTO_F64

    def pack(self, out, rows):
        torch = _torch()
        buf = torch.empty((rows.numel(), out.shape[1]), dtype=out.dtype, device=out.device)
        _lib.check(self.lib.alto_pack_rows(out.data_ptr(), self._dt(out), rows.data_ptr(), rows.numel(),
                                           out.shape[1], buf.data_ptr(), _lib.stream_ptr()), "alto_pack_rows")
        return buf

    def unpack(self, out, rows, buf):
        _lib.check(self.lib.alto_unpack_rows(out.data_ptr(), self._dt(out), rows.data_ptr(), rows.numel(),
                                             out.shape[1], buf.data_ptr(), _lib.stream_ptr()), "alto_unpack_rows")

    def add_rows(self, out, rows, buf):
        _lib.check(self.lib.alto_add_rows(out.data_ptr(), self._dt(out), rows.data_ptr(), rows.numel(),
                                          out.shape[1], buf.data_ptr(), _lib.stream_ptr()), "alto_add_rows")

    def hadamard(self, grams, skip):
        from .cpd import hadamard_device

        return hadamard_device(grams, skip)

    def solve(self, v, m):
        torch = _torch()
        x = torch.empty_like(m)
        self.ws.status.zero_()
        _lib.check(self.lib.alto_solve_rows(v.data_ptr(), m.data_ptr(), m.shape[0], m.shape[1], x.data_ptr(),
                                            self.ws.status.data_ptr(), self.ws.buf.data_ptr(), self.ws.bytes,
                                            _lib.stream_ptr()), "alto_solve_rows")
        if int(self.ws.status.item()) == 2:
            raise np.linalg.LinAlgError("normal equations singular even with ridge")
        return x

    def colsumsq(self, x, mask):
        torch = _torch()
        out = torch.empty(x.shape[1], dtype=torch.float64, device=x.device)
        _lib.check(self.lib.alto_colsumsq(x.data_ptr(), x.shape[0], x.shape[1], mask.data_ptr(), out.data_ptr(),
                                          self.ws.buf.data_ptr(), self.ws.bytes, _lib.stream_ptr()), "alto_colsumsq")
        return out

    def normalize(self, x, colsumsq, x32=None):
        torch = _torch()
        lam = torch.empty(x.shape[1], dtype=torch.float64, device=x.device)
        _lib.check(self.lib.alto_normalize(x.data_ptr(), None if x32 is None else x32.data_ptr(), x.shape[0],
                                           x.shape[1], colsumsq.data_ptr(), lam.data_ptr(),
                                           self.ws.status.data_ptr(), _lib.stream_ptr()), "alto_normalize")
        return lam

    def gram(self, f, mask=None):
        torch = _torch()
        g = torch.empty((f.shape[1], f.shape[1]), dtype=torch.float64, device=f.device)
        _lib.check(self.lib.alto_gram_masked(f.data_ptr(), self._dt(f), f.shape[0], f.shape[1],
                                             None if mask is None else mask.data_ptr(), g.data_ptr(),
                                             self.ws.buf.data_ptr(), self.ws.bytes, _lib.stream_ptr()),
                   "alto_gram_masked")
        return g

    def fit_inner(self, m, f, lam, mask):
        torch = _torch()
        out = torch.empty(1, dtype=torch.float64, device=m.device)
        _lib.check(self.lib.alto_fit_inner_masked(m.data_ptr(), f.data_ptr(), lam.data_ptr(), m.shape[0], m.shape[1],
                                                  mask.data_ptr(), out.data_ptr(), self.ws.buf.data_ptr(),
                                                  self.ws.bytes, _lib.stream_ptr()), "alto_fit_inner_masked")
        return out

    def sumsq(self):
        torch = _torch()
        from .cpd import sumsq_device

        return torch.tensor([sumsq_device(self.shard.vals, self.ws)], dtype=torch.float64, device=self.dev)

    def to_gather(self, f64):
        """Factor copy the MTTKRP gathers from (float32 for float32 shards)."""
        torch = _torch()
        return f64.float() if self.shard.vals.dtype == torch.float32 else f64


class ShardedCpAls:
    """CP-ALS over key-range shards (one per rank), see module docstring."""

    def __init__(self, ops, dims, rank: int, seed: int = 0, group=None, init_factors=None):
        torch = _torch()
        self.ops = ops
        self.dims = tuple(int(d) for d in dims)
        self.rank = rank
        self.group = group
        if init_factors is None:
            rng = np.random.default_rng(seed)  # the reference's init draw (cpd.py:206-208)
            init_factors = [rng.random((d, rank)) for d in self.dims]
        dev = ops.dev
        self.f64 = [torch.as_tensor(np.asarray(f, dtype=np.float64)).to(dev) for f in init_factors]
        self.fg = [ops.to_gather(f) for f in self.f64]
        self.plans = [ShardRows(ops.touched_rows(n), group) for n in range(len(self.dims))]
        # initial factors are identical on all ranks: their Grams need no reduction
        self.grams = [ops.gram(f) for f in self.f64]
        self.lam = torch.ones(rank, dtype=torch.float64, device=dev)
        ns = ops.sumsq()
        self._all_reduce(ns)
        self.norm_sq = float(ns.item())

    def _all_reduce(self, t):
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def mttkrp(self, mode: int):
        out = self.ops.mttkrp(self.fg, mode)
        exchange_shared(out, self.plans[mode], self.ops)
        return out

    def fit(self, m, mode: int) -> float:
        if self.norm_sq == 0.0:
            return 1.0
        inner = self._all_reduce(self.ops.fit_inner(m, self.f64[mode], self.lam, self.plans[mode].mask))
        vall = self.ops.hadamard(self.grams, None)
        lam = self.lam.double()
        model_sq = float((lam @ vall @ lam).item())
        resid = max(self.norm_sq - 2.0 * float(inner.item()) + model_sq, 0.0)
        return 1.0 - math.sqrt(resid) / math.sqrt(self.norm_sq)

    def update(self, mode: int):
        m = self.mttkrp(mode)
        v = self.ops.hadamard(self.grams, mode)
        x = self.ops.solve(v, m)
        sq = self._all_reduce(self.ops.colsumsq(x, self.plans[mode].mask))
        self.lam = self.ops.normalize(x, sq)
        self.f64[mode] = x
        self.fg[mode] = self.ops.to_gather(x)
        self.grams[mode] = self._all_reduce(self.ops.gram(x, self.plans[mode].mask))
        return m

    def run(self, max_iters: int, tol: float = 0.0):
        m0 = self.mttkrp(0)
        hist = [self.fit(m0, 0)]
        iters = 0
        for _ in range(max_iters):
            for mode in range(len(self.dims)):
                m = self.update(mode)
            hist.append(self.fit(m, len(self.dims) - 1))
            iters += 1
            if abs(hist[-1] - hist[-2]) < tol:
                break
        return hist, iters

    def gather_factors(self):
        """Full factors: each row contributed by its owner, summed across ranks."""
        torch = _torch()
        full = []
        for n, f in enumerate(self.f64):
            own = f * self.plans[n].owned.to(f.dtype)[:, None]
            full.append(self._all_reduce(own.clone()))
        return full
