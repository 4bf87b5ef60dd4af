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
