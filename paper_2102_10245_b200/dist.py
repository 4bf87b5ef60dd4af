"""Key-range-sharded MTTKRP / CP-ALS across GPUs.

The reference has no distributed path (threads only, mttkrp.py:120-129; the
paper lists distributed memory as future work).  Here each rank
(one process per GPU, torch.distributed over NCCL) holds one contiguous
key range of the sorted ALTO stream — exactly an ALTO partition
(format.py:127-154) — and full-size factor matrices.

Per mode n:
  1. local MTTKRP over the shard (rows touched only by this shard are final);
  2. shared-row reduction: rows touched by >= 2 shards are packed into one
     compact buffer and summed with a single all-reduce (volume = shared
     rows x R, not I_n x R);
  3. every rank solves the rows it touches (X V = M); rows shared between
     shards are solved redundantly by each toucher, so no factor rows need to
     be sent back;
  4. column norms, the Gram of the new factor and the fit inner product are
     reduced over *owned* rows only (rows touched by exactly one shard, and
     shared rows owned by their lowest-rank toucher) — R, R x R and 1 values
     per mode cross the interconnect.

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


class ShardRows:
    """Exchange plan of one mode: shared rows and this rank's owned-row mask."""

    def __init__(self, touched, group=None):
        torch = _torch()
        import torch.distributed as dist

        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        cnt = touched.to(torch.int32)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
        first = torch.where(touched, torch.full_like(cnt, rank), torch.full_like(cnt, world))
        dist.all_reduce(first, op=dist.ReduceOp.MIN, group=group)
        self.shared_rows = torch.nonzero(cnt >= 2).flatten().to(torch.int64)
        self.owned = touched & ((cnt == 1) | (first == rank))
        self.mask = self.owned.to(torch.uint8)
        self.touched = touched
        self.group = group

    @property
    def n_shared(self) -> int:
        return int(self.shared_rows.numel())


def reduce_shared(out, plan: ShardRows, ops) -> None:
    """Sum the partial rows of `out` that several shards touch (in place)."""
    import torch.distributed as dist

    if plan.n_shared == 0:
        return
    buf = ops.pack(out, plan.shared_rows)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=plan.group)
    ops.unpack(out, plan.shared_rows, buf)


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
        from .mttkrp import row_index

        _perm, ptr = row_index(self.shard, mode)
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
        reduce_shared(out, self.plans[mode], self.ops)
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
