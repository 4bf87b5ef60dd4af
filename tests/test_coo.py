"""COO ingestion: device coalesce bitwise against the
reference semantics (oracle.coalesce, coo.py:97-114), the text format
(pkg/tests/test_coo.py cases), and the reference sampler's pinned count."""

import io

import numpy as np
import pytest

from oracle import alto_oracle as orc


class TestParseErrors:
    """Malformed text is rejected on the host before any device work (CPU)."""

    @pytest.mark.parametrize("text,match", [
        ("# dims: 4 x 2\n1 1 1 1.0", "dims header"),
        ("# dims: 4 0 2\n1 1 1 1.0", "positive"),
        ("1 1 1 1.0\n1 1 1.0", "line 2"),
        ("1 x 1 1.0", "malformed"),
        ("0 1 1 1.0", "one-based"),
        ("# only a comment\n", "no data"),
        ("7\n", "at least one index"),
    ])
    def test_errors(self, at, text, match):
        with pytest.raises(at.TnsParseError, match=match):
            at.parse_tns(text)

    def test_override_errors(self, at):
        with pytest.raises(at.TnsParseError, match="exceeds"):
            at.parse_tns("3 1 1.0", dims=(2, 2))
        with pytest.raises(at.TnsParseError, match="modes"):
            at.parse_tns("1 1 1.0", dims=(2, 2, 2))
        with pytest.raises(at.TnsParseError, match="exceeds"):
            at.parse_tns("# dims: 2 2\n3 1 1.0")

    def test_is_value_error(self, at):
        assert issubclass(at.TnsParseError, ValueError)

    def test_write_format(self, at):
        assert at.write_tns(at.CooTensor((1, 1, 1), [[0, 0, 0]], [2.0])) == "# dims: 1 1 1\n1 1 1 2.0\n"
        buf = io.StringIO()
        assert at.write_tns(at.CooTensor((2, 2), [[1, 0]], [0.5]), buf) is None
        assert buf.getvalue() == "# dims: 2 2\n2 1 0.5\n"


@pytest.mark.gpu
class TestDeviceCoalesce:
    @pytest.mark.parametrize("dims,m,seed", [((4, 4), 40, 0), ((50, 40, 30), 20000, 1),
                                             ((7, 3, 5, 2, 4), 5000, 2), ((1 << 40, 1 << 40, 1 << 30), 3000, 3),
                                             ((1, 9), 50, 4), ((3,), 100, 5)])
    def test_bitwise_vs_reference_semantics(self, at, dims, m, seed):
        from paper_2102_10245_b200.coo import coalesce_device

        rng = np.random.default_rng(seed)
        hi = np.minimum(np.asarray(dims), 6)  # many duplicates, also on huge modes
        c = rng.integers(0, hi, size=(m, len(dims)), dtype=np.int64)
        if max(dims) > 1 << 20:
            c[::3] = rng.integers(0, dims, size=(len(c[::3]), len(dims)), dtype=np.int64)
        v = rng.standard_normal(m) * 10.0 ** rng.integers(-8, 8, m)
        v[::7] = -0.0
        rc, rv = orc.coalesce(c, v)
        oc, ov = coalesce_device(dims, c, v)
        assert np.array_equal(oc.cpu().numpy(), rc)
        assert np.array_equal(ov.cpu().numpy().view(np.uint64), rv.view(np.uint64))

    def test_coo_coalesce_api(self, at):
        t = at.CooTensor((4, 4), [[2, 1], [0, 3], [2, 1]], [1.0, 2.0, 5.0]).coalesce()
        assert t.coords.tolist() == [[0, 3], [2, 1]]
        assert t.values.tolist() == [2.0, 6.0]

    def test_random_tensor_pinned(self, at):
        """The reference sampler's frozen count (pkg/tests/test_coo.py:136-139)."""
        assert at.random_tensor((50, 40, 30), 10000, seed=7).nnz == 9228
        a = at.random_tensor((9, 9, 9), 200, seed=3)
        assert a.isequal(at.random_tensor((9, 9, 9), 200, seed=3))

    def test_large_property(self):
        """5M rows drawn from a small box: sums of the coalesced tensor equal the
        input's (size-independent), rows strictly increasing, bitwise = oracle."""
        from paper_2102_10245_b200.coo import coalesce_device

        rng = np.random.default_rng(11)
        dims = (300, 200, 100)
        c = rng.integers(0, dims, size=(5_000_000, 3), dtype=np.int64)
        v = rng.random(5_000_000)
        oc, ov = coalesce_device(dims, c, v)
        oc, ov = oc.cpu().numpy(), ov.cpu().numpy()
        key = (oc[:, 0] * 200 + oc[:, 1]) * 100 + oc[:, 2]
        assert (np.diff(key) > 0).all()
        rc, rv = orc.coalesce(c, v)
        assert np.array_equal(oc, rc) and np.array_equal(ov, rv)


@pytest.mark.gpu
class TestParseTns:
    def test_cases(self, at):
        t = at.parse_tns("1 1 1 2.0")
        assert t.dims == (1, 1, 1) and t.coords.tolist() == [[0, 0, 0]] and t.values.tolist() == [2.0]
        t = at.parse_tns("1 2 1 1.0\n1 2 1 3.5")
        assert t.nnz == 1 and t.values.tolist() == [4.5]
        t = at.parse_tns("# header\n\n  2 3 1.5\n# trailing\n1 1 -2\n")
        assert t.dims == (2, 3) and t.nnz == 2
        assert at.parse_tns("4 8 2 1.0\n1 1 1 1.0").dims == (4, 8, 2)
        assert at.parse_tns("1 1 1 1.0", dims=(4, 8, 2)).dims == (4, 8, 2)
        assert at.parse_tns("# dims: 4 8 2\n2 1 1 1.0").dims == (4, 8, 2)
        assert at.parse_tns("# dims: 4 8 2\n2 1 1 1.0", dims=(5, 9, 3)).dims == (5, 9, 3)
        assert at.parse_tns("2 1 1 1.0\n# dims: 4 8 2\n").dims == (2, 1, 1)
        t = at.parse_tns("# dims: 4 8 2\n")
        assert t.dims == (4, 8, 2) and t.nnz == 0
        assert at.parse_tns(io.StringIO("2 2 7.0")).dims == (2, 2)

    def test_round_trip_exact(self, at):
        t = at.random_tensor((30, 20, 10), 1000, seed=5)
        back = at.parse_tns(at.write_tns(t))
        assert back.dims == t.dims
        assert np.array_equal(back.coords, t.coords) and np.array_equal(back.values, t.values)
        e = at.CooTensor((3, 3), np.empty((0, 2)), np.empty(0))
        assert at.write_tns(e) == "# dims: 3 3\n"
        assert at.parse_tns(at.write_tns(e)).nnz == 0
        assert at.parse_tns(at.write_tns(at.CooTensor((4, 8, 2), [[1, 6, 1]], [6.0]))).dims == (4, 8, 2)


def _golden():
    import os

    from conftest import GOLDEN

    return np.load(os.path.join(GOLDEN, "coo_coalesce.npz"))


def test_oracle_pinned_to_reference():
    """oracle.coalesce reproduces the reference's outputs bitwise (CPU)."""
    g = _golden()
    for k in range(4):
        c, v = orc.coalesce(g[f"in_coords{k}"], g[f"in_values{k}"])
        assert np.array_equal(c, g[f"coords{k}"])
        assert np.array_equal(v.view(np.uint64), g[f"values{k}"].view(np.uint64))


@pytest.mark.gpu
def test_device_coalesce_golden(at):
    """Device coalesce against the reference's own outputs, and random_tensor
    against the reference's sampler output (coordinates and values)."""
    from paper_2102_10245_b200.coo import coalesce_device

    g = _golden()
    for k in range(4):
        oc, ov = coalesce_device(tuple(int(x) for x in g[f"dims{k}"]), g[f"in_coords{k}"], g[f"in_values{k}"])
        assert np.array_equal(oc.cpu().numpy(), g[f"coords{k}"])
        assert np.array_equal(ov.cpu().numpy().view(np.uint64), g[f"values{k}"].view(np.uint64))
    r = at.random_tensor((50, 40, 30), 10000, seed=7)
    assert np.array_equal(r.coords, g["rand_coords"]) and np.array_equal(r.values, g["rand_values"])
