"""Multi-process (world_size 2, gloo, CPU) tests of the key-range-sharded
MTTKRP / CP-ALS exchange logic (paper_2102_10245_b200/dist.py).

The per-shard compute is injected as CPU ops built on the oracle, so these
tests exercise exactly the distributed part — shard plans, the owner-directed
shared-row exchange (grouped send/recv), owner-masked reductions — and compare against the single-process
oracle (the reference algorithm).
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import alto_oracle as orc
from paper_2102_10245_b200 import synth


class CpuOps:
    """Oracle-backed stand-in for dist.DeviceOps (test infrastructure)."""

    def __init__(self, lay, words, vals):
        self.lay, self.words, self.vals = lay, words, vals
        self.coords = orc.decode(lay, words)
        self.dev = torch.device("cpu")

    def touched_rows(self, mode):
        t = torch.zeros(self.lay.dims[mode], dtype=torch.bool)
        if len(self.coords):
            t[torch.from_numpy(self.coords[:, mode])] = True
        return t

    def mttkrp(self, factors, mode):
        f = [x.numpy() for x in factors]
        return torch.from_numpy(orc.mttkrp_seq(self.lay, self.words, self.vals, f, mode))

    def pack(self, out, rows):
        return out.index_select(0, rows).contiguous()

    def unpack(self, out, rows, buf):
        out.index_copy_(0, rows, buf)

    def add_rows(self, out, rows, buf):
        out.index_add_(0, rows, buf)

    def hadamard(self, grams, skip):
        v = torch.ones_like(grams[0])
        for n, g in enumerate(grams):
            if n != skip:
                v = v * g
        return v

    def solve(self, v, m):
        return torch.from_numpy(orc.solve(v.numpy(), m.numpy()))

    def colsumsq(self, x, mask):
        return (x * x * mask.to(x.dtype)[:, None]).sum(0)

    def normalize(self, x, sq):
        lam = torch.sqrt(sq)
        x /= torch.where(lam == 0, torch.ones_like(lam), lam)
        return lam

    def gram(self, f, mask=None):
        g = f if mask is None else f * mask.to(f.dtype)[:, None]
        return g.T @ g

    def fit_inner(self, m, f, lam, mask):
        return (m * f * lam[None, :] * mask.to(m.dtype)[:, None]).sum().reshape(1)

    def sumsq(self):
        return torch.tensor([float(np.dot(self.vals, self.vals))], dtype=torch.float64)

    def to_gather(self, f):
        return f


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_10245_b200.dist import ShardedCpAls, ShardRows

        dims, nnz, rank_r, iters = case
        st = synth.make_tensor(synth.SynthConfig("cfg8", dims, nnz, (("zipf", 1.1),) * len(dims), "uniform01",
                                                 "float64", rank_r), nnz=nnz, seed=77)
        lay = orc.build_layout(dims)
        words, vals = orc.build(lay, st.coords, st.values)
        offs = orc.offsets_for(words.shape[0], world)
        a, b = int(offs[rank]), int(offs[rank + 1])
        ops = CpuOps(lay, words[a:b], vals[a:b])
        solver = ShardedCpAls(ops, dims, rank_r, seed=3)
        # exchange plan: shared rows == rows touched by >= 2 shards
        coords = orc.decode(lay, words)
        for n, plan in enumerate(solver.plans):
            seen = [set(coords[offs[r]:offs[r + 1], n].tolist()) for r in range(world)]
            shared = sorted({x for r in range(world) for x in seen[r]
                             if sum(x in s for s in seen) >= 2})
            assert plan.shared_rows.tolist() == shared
            owned = dist_owned = plan.owned.to(torch.int32)
            dist.all_reduce(dist_owned)
            touched_any = np.zeros(dims[n], dtype=np.int32)
            touched_any[coords[:, n]] = 1
            assert dist_owned.numpy().tolist() == touched_any.tolist()  # every touched row owned exactly once
            del owned
            # owner-directed lists: rank r sends exactly the shared rows it touches
            # but does not own, each to its owner (the lowest-rank toucher)
            mine = sorted(x for x in seen[rank] if x in set(shared))
            want = {}
            for x in mine:
                o = min(r for r in range(world) if x in seen[r])
                if o != rank:
                    want.setdefault(o, []).append(x)
            assert {o: r.tolist() for o, r in plan.send.items()} == want
            got_recv = {r: v.tolist() for r, v in plan.recv.items()}
            exp_recv = {r: sorted(x for x in seen[r] if x in set(shared) and x in seen[rank]
                                  and min(q for q in range(world) if x in seen[q]) == rank)
                        for r in range(world) if r != rank}
            assert got_recv == {r: v for r, v in exp_recv.items() if v}
        # one sharded MTTKRP with the shared-row reduction == the global one
        m = solver.mttkrp(1)
        ref = orc.mttkrp_seq(lay, words, vals, [f.numpy() for f in solver.f64], 1)
        touched = solver.plans[1].touched.numpy()
        assert np.allclose(m.numpy()[touched], ref[touched], rtol=1e-12, atol=1e-12)
        hist, _ = solver.run(iters)
        full = solver.gather_factors()
        if rank == 0:
            np.save(os.path.join(outdir, "hist.npy"), np.asarray(hist))
            for n, f in enumerate(full):
                np.save(os.path.join(outdir, f"f{n}.npy"), f.numpy())
            np.save(os.path.join(outdir, "lam.npy"), solver.lam.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [(((60, 50, 40), 6000, 4, 3), 2), (((30, 20, 25, 15), 4000, 3, 2), 2),
                                        (((60, 50, 40), 6000, 4, 2), 3)])
def test_sharded_cpals_matches_single_process(case, world):
    dims, nnz, rank_r, iters = case
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), case, d), nprocs=world, join=True)
        hist = np.load(os.path.join(d, "hist.npy"))
        st = synth.make_tensor(synth.SynthConfig("cfg8", dims, nnz, (("zipf", 1.1),) * len(dims), "uniform01",
                                                 "float64", rank_r), nnz=nnz, seed=77)
        lay = orc.build_layout(dims)
        words, vals = orc.build(lay, st.coords, st.values)
        f, w, ref_hist, _ = orc.cpd_als(lay, words, vals, rank_r, max_iters=iters, tol=0.0, seed=3)
        np.testing.assert_allclose(hist, ref_hist, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(np.load(os.path.join(d, "lam.npy")), w, rtol=1e-9)
        for n in range(len(dims)):
            np.testing.assert_allclose(np.load(os.path.join(d, f"f{n}.npy")), f[n], rtol=1e-8, atol=1e-10)
