"""Device ops of the key-range-sharded CP-ALS (dist.DeviceOps) on one B200,
world_size 1 over NCCL: pack/unpack kernels and the masked reductions, and a
full ShardedCpAls run against the single-device CP-ALS."""

import os
import socket

import numpy as np
import pytest

from paper_2102_10245_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group():
    import torch.distributed as dist

    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1)
    yield None
    dist.destroy_process_group()


def test_pack_unpack_rows(at):
    import torch

    from paper_2102_10245_b200.dist import DeviceOps

    alto = at.build_alto(at.random_tensor((40, 30, 20), 2000, seed=1))
    ops = DeviceOps(alto, 16)
    for dt in (torch.float32, torch.float64):
        out = torch.randn(40, 16, dtype=dt, device="cuda")
        rows = torch.tensor([0, 3, 17, 39], dtype=torch.int64, device="cuda")
        buf = ops.pack(out, rows)
        assert torch.equal(buf, out[rows])
        ops.unpack(out, rows, buf * 2)
        assert torch.equal(out[rows], buf * 2)


def test_sharded_world1_matches_device_cpals(at, group):
    import torch

    from paper_2102_10245_b200.dist import DeviceOps, ShardedCpAls

    st = synth.make_tensor(2, nnz=200_000)
    alto = at.build_alto(at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64)))
    solver = ShardedCpAls(DeviceOps(alto, 8), st.config.dims, 8, seed=5)
    hist, _ = solver.run(3)
    ref = at.cpd_als(alto, rank=8, max_iters=3, tol=0.0, seed=5, backend="atomic", partitions=4)
    np.testing.assert_allclose(hist, ref.fit_history, rtol=1e-9, atol=1e-12)
    full = solver.gather_factors()
    for f, g in zip(full, ref.factors):
        np.testing.assert_allclose(f.cpu().numpy(), g, rtol=1e-6, atol=1e-9)


def _gpu_worker(rank, world, port, outdir):
    """One rank of the 2-rank sharded CP-ALS on cuda:0 (gloo: the box has one
    GPU; the kernels of the two ranks never wait on each other on the device,
    the exchange goes through the host)."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_10245_b200.dist import DeviceOps, ShardedCpAls, build_shard
        from paper_2102_10245_b200.layout import build_masks

        st = synth.make_tensor(2, nnz=200_000)
        dims = st.config.dims
        coords = torch.from_numpy(st.coords).cuda()
        vals = torch.from_numpy(st.values.astype(np.float64)).cuda()
        shard, info = build_shard(build_masks(dims), coords, vals, rank, world, 8)
        solver = ShardedCpAls(DeviceOps(shard, 8), dims, 8, seed=5)
        hist, _ = solver.run(3)
        full = solver.gather_factors()
        nnz = torch.tensor([shard.nnz], dtype=torch.int64)
        dist.all_reduce(nnz)
        if rank == 0:
            np.save(os.path.join(outdir, "hist.npy"), np.asarray(hist))
            np.save(os.path.join(outdir, "nnz.npy"), nnz.numpy())
            for n, f in enumerate(full):
                np.save(os.path.join(outdir, f"f{n}.npy"), f.cpu().numpy())
        # the shard is exactly this rank's key range of the global sorted stream
        keys = shard.indices
        np.save(os.path.join(outdir, f"keys{rank}.npy"), keys)
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_cpals_on_device(at, tmp_path):
    """ShardedCpAls with DeviceOps over 2 ranks (cost-balanced key-range
    shards built per rank, owner-directed exchange) == single-device cpd_als."""
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_gpu_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    st = synth.make_tensor(2, nnz=200_000)
    alto = at.build_alto(at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64)))
    assert int(np.load(tmp_path / "nnz.npy")[0]) == alto.nnz
    k0, k1 = np.load(tmp_path / "keys0.npy"), np.load(tmp_path / "keys1.npy")
    assert np.array_equal(np.concatenate([k0, k1]), alto.indices)  # contiguous key ranges, in order
    ref = at.cpd_als(alto, rank=8, max_iters=3, tol=0.0, seed=5, backend="atomic", partitions=4)
    np.testing.assert_allclose(np.load(tmp_path / "hist.npy"), ref.fit_history, rtol=1e-9, atol=1e-12)
    for n, g in enumerate(ref.factors):
        np.testing.assert_allclose(np.load(tmp_path / f"f{n}.npy"), g, rtol=1e-6, atol=1e-9)
