"""Pin the full-size C oracle (oracle/mttkrp_oracle.c) against fixtures the
reference produced (tests/golden/make_golden.py runs the unmodified
reference's mttkrp_oracle, mttkrp.py:64-77) and against the NumPy
restatement.  CPU only: the C oracle is what the full-size GPU parity tests
(tests/test_gpu_fullsize.py) compare against."""

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden
from oracle import alto_oracle as orc
from oracle import oracle_c
from test_oracle_golden import _factors, _inputs


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_c_oracle_bitwise_vs_reference_goldens(name):
    data, meta = load_golden(name)
    if not meta["with_mttkrp"]:
        pytest.skip("fixture has no MTTKRP outputs")
    coords, values = _inputs(data, meta)
    factors = _factors(data, meta)
    u = np.random.default_rng(99).random(meta["rank"])
    for mode in range(len(meta["dims"])):
        out = oracle_c.mttkrp_coo(coords, values, factors, mode, threads=4)
        key = f"m{mode}_oracle"
        if meta.get("project"):
            assert np.array_equal(out @ u, data[key + "_proj"]), key
            assert np.linalg.norm(out) == float(data[key + "_fro"]) or \
                abs(np.linalg.norm(out) - float(data[key + "_fro"])) <= 1e-15 * float(data[key + "_fro"])
        else:
            assert np.array_equal(out, data[key]), key


@pytest.mark.parametrize("order,rank", [(3, 16), (4, 32), (5, 16), (3, 7), (1, 4), (2, 3)])
def test_c_oracle_equals_numpy_and_thread_count_invariant(order, rank):
    rng = np.random.default_rng(order * 100 + rank)
    dims = tuple(int(x) for x in rng.integers(3, 40, size=order))
    m = 20000
    coords = np.stack([rng.integers(0, d, m) for d in dims], 1)
    # skewed rows: many elements in a few rows (input order matters bitwise)
    coords[: m // 2, 0] = rng.integers(0, 2, m // 2)
    vals32 = rng.random(m).astype(np.float32)
    factors = [rng.random((d, rank)).astype(np.float32).astype(np.float64) for d in dims]
    for mode in range(order):
        ref = orc.mttkrp_coo(coords, vals32.astype(np.float64), factors, mode)
        for t in (1, 2, 8):
            out = oracle_c.mttkrp_coo(coords, vals32, factors, mode, threads=t)
            assert np.array_equal(out, ref), (mode, t)


def test_c_oracle_errors_and_rel_error():
    f = [np.ones((3, 2)), np.ones((4, 2))]
    with pytest.raises(ValueError):
        oracle_c.mttkrp_coo(np.array([[3, 0]]), np.ones(1), f, 0)
    a = np.arange(12, dtype=np.float64).reshape(6, 2)
    b = a.copy()
    b[0, 0] += 1.0
    assert oracle_c.rel_error(a, a) == 0.0
    assert abs(oracle_c.rel_error(b, a) - 1.0 / np.linalg.norm(a)) < 1e-15
    assert abs(oracle_c.rel_error(b.astype(np.float32), a) - 1.0 / np.linalg.norm(a)) < 1e-12
    empty = oracle_c.mttkrp_coo(np.zeros((0, 2), dtype=np.int64), np.zeros(0), f, 1)
    assert empty.shape == (4, 2) and not empty.any()
