"""K8/K9 pull engine (csrc/alto_pull.cuh): slice interval buffers + the
deterministic pull (Buffered, reference mttkrp.py:132-175) and the on-the-fly
boundary-flag Atomic scheme (mttkrp.py:178-224), against the C oracle
(bitwise restatement of mttkrp_oracle, mttkrp.py:64-77)."""

import numpy as np
import pytest

from oracle import oracle_c
from paper_2102_10245_b200 import synth

pytestmark = pytest.mark.gpu

WIDE = synth.SynthConfig("cfg9", (1 << 22, 1 << 22, 1 << 21), 0, (("zipf", 1.05),) * 3, "uniform01", "float32", 16)


def _tensor(at, cfg, nnz, dtype):
    st = synth.make_tensor(WIDE if cfg == "wide" else cfg, nnz=nnz)
    alto = at.build_alto(at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64)), dtype=dtype)
    return st, alto


@pytest.mark.parametrize("cfg,nnz", [(2, 300_000), (4, 200_000), (3, 150_000), ("wide", 200_000), (1, 100_000)])
@pytest.mark.parametrize("combo", ["f32/f32/f32", "f32/f32/f64", "f64/f64/f64", "f32/f64/f64"])
@pytest.mark.parametrize("atomic", [False, True])
def test_pull_vs_oracle(at, cfg, nnz, combo, atomic):
    import torch

    from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_pull

    vd, fd, od = combo.split("/")
    st, alto = _tensor(at, cfg, nnz, "float32" if vd == "f32" else "float64")
    dims = st.config.dims
    rank = 32 if cfg == 3 else 16
    rng = np.random.default_rng(11)
    fac = [rng.random((d, rank)).astype(np.float32).astype(np.float64 if fd == "f64" else np.float32) for d in dims]
    fdev = factors_to_device(fac)
    vals = st.values.astype(np.float32) if vd == "f32" else st.values.astype(np.float64)
    tol = 1e-5 if (fd == "f32" or od == "f32") else 1e-12
    for mode in range(len(dims)):
        ref = oracle_c.mttkrp_coo(st.coords, vals, [f.astype(np.float64) for f in fac], mode)
        out = torch.full((dims[mode], rank), float("nan"), dtype=torch.float32 if od == "f32" else torch.float64,
                         device="cuda")
        got = mttkrp_pull(alto, fdev, mode, out=out, atomic=atomic)
        assert got is not None, (cfg, combo, atomic)
        g = got.cpu().numpy()
        assert not np.isnan(g).any(), "every output row must be written (zero fill)"
        assert oracle_c.rel_error(g, ref) <= tol, (cfg, combo, atomic, mode, oracle_c.rel_error(g, ref))


@pytest.mark.parametrize("rank", [8, 16, 32, 64])
@pytest.mark.parametrize("order", [3, 4, 5])
def test_pull_ranks_orders(at, rank, order):
    """Every instantiated (order, rank) on a skewed tensor with empty rows at
    both ends and a head row spanning many slices."""
    import torch

    from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_pull

    rng = np.random.default_rng(rank * 10 + order)
    dims = tuple(int(x) for x in rng.integers(20, 300, size=order))
    m = 40_000
    coords = np.stack([rng.integers(2, d - 2, m) for d in dims], 1)
    coords[: m // 3, 0] = 5  # one row holds a third of the tensor
    coords = np.unique(coords, axis=0)
    rng.shuffle(coords)
    vals = rng.random(coords.shape[0]).astype(np.float32)
    alto = at.build_alto(at.CooTensor(dims, coords, vals.astype(np.float64)), dtype="float32")
    fac = [rng.random((d, rank)).astype(np.float32) for d in dims]
    fdev = factors_to_device(fac)
    for mode in range(order):
        ref = oracle_c.mttkrp_coo(coords, vals, [f.astype(np.float64) for f in fac], mode)
        got = mttkrp_pull(alto, fdev, mode, out_dtype=torch.float32)
        assert got is not None
        assert oracle_c.rel_error(got.cpu().numpy(), ref) <= 1e-6, (rank, order, mode)


def test_pull_bitwise_deterministic(at):
    from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_pull

    st, alto = _tensor(at, 2, 400_000, "float32")
    rng = np.random.default_rng(3)
    fdev = factors_to_device([rng.random((d, 16)) for d in st.config.dims])  # float64 factors
    for mode in range(3):
        a = mttkrp_pull(alto, fdev, mode).cpu().numpy()
        b = mttkrp_pull(alto, fdev, mode).cpu().numpy()
        assert np.array_equal(a, b)


def test_pull_single_row_and_tiny(at):
    """All elements in one output row (every slice shares it) and tensors
    smaller than one slice."""
    from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_pull

    rng = np.random.default_rng(5)
    for dims, m in [((7, 300, 200), 50_000), ((9, 8, 7), 5), ((9, 8, 7), 1), ((3, 1000, 1000), 30_000)]:
        coords = np.stack([rng.integers(0, d, m * 2) for d in dims], 1)
        coords[:, 0] = 0 if dims[0] == 7 else coords[:, 0]
        coords = np.unique(coords, axis=0)[:m]
        vals = rng.random(coords.shape[0])
        alto = at.build_alto(at.CooTensor(dims, coords, vals))
        fac = [rng.random((d, 16)) for d in dims]
        fdev = factors_to_device(fac)
        for mode in range(3):
            ref = oracle_c.mttkrp_coo(coords, vals, fac, mode)
            for atomic in (False, True):
                got = mttkrp_pull(alto, fdev, mode, atomic=atomic).cpu().numpy()
                assert oracle_c.rel_error(got, ref) <= 1e-12, (dims, m, mode, atomic)
