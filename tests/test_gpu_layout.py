"""Device codecs (K1 linearize, K4 delinearize) against the reference's
goldens (pkg/tests/test_layout.py) and the oracle."""

import math

import numpy as np
import pytest

from oracle import alto_oracle as orc

pytestmark = pytest.mark.gpu


def deposit(layout, coords) -> int:
    """Mask-only deposit (pkg/tests/test_layout.py:12-25 idea)."""
    pos = 0
    for n, c in enumerate(coords):
        g = 0
        for p in range(layout.width):
            if (layout.masks[n] >> p) & 1:
                pos |= ((int(c) >> g) & 1) << p
                g += 1
    return pos


class TestLinearize:
    def test_worked_example(self, at):
        lay = at.build_masks((4, 8, 2))
        for coords, want in {(1, 0, 0): 2, (0, 3, 0): 20, (2, 2, 1): 25, (1, 6, 1): 51, (0, 0, 0): 0}.items():
            assert at.linearize(lay, coords) == want

    def test_golden_232(self, at):
        lay = at.build_masks((5, 3, 7))
        assert at.linearize(lay, (4, 2, 6)) == 232

    def test_matches_deposit(self, at):
        rng = np.random.default_rng(42)
        for dims in [(4, 8, 2), (5, 3, 7), (1, 9, 1, 16), (600, 2, 45)]:
            lay = at.build_masks(dims)
            coords = rng.integers(0, dims, size=(64, len(dims)))
            words = at.linearize_array(lay, coords)
            for row, w in zip(coords, words):
                assert int(w[0]) == deposit(lay, row)

    def test_out_of_range(self, at):
        lay = at.build_masks((4, 8, 2))
        for bad in [(4, 0, 0), (0, -1, 0)]:
            with pytest.raises(ValueError):
                at.linearize(lay, bad)
        with pytest.raises(ValueError):
            at.linearize(lay, (0, 0))
        with pytest.raises(ValueError):
            at.linearize_array(lay, np.array([[0, 0, 5]]))
        with pytest.raises(ValueError):
            at.linearize_array(lay, np.zeros((3, 2), dtype=np.int64))

    def test_monotone(self, at):
        lay = at.build_masks((5, 3, 7))
        for n, dim in enumerate(lay.dims):
            probes = np.tile(np.array([2, 1, 3]), (dim, 1))
            probes[:, n] = np.arange(dim)
            w = at.linearize_array(lay, probes)[:, 0]
            assert list(w) == sorted(w) and len(set(w.tolist())) == dim


class TestDelinearize:
    def test_worked_and_flags_ignored(self, at):
        lay = at.build_masks((4, 8, 2))
        assert at.delinearize(lay, 25) == (2, 2, 1)
        assert at.delinearize(lay, 25 | (1 << 6)) == (2, 2, 1)
        assert at.delinearize(lay, 25 | (1 << 63)) == (2, 2, 1)

    def test_singleton_modes(self, at):
        lay = at.build_masks((1, 9, 1, 16))
        words = np.arange(10, dtype=np.uint64)[:, None]
        c = at.delinearize_array(lay, words)
        assert (c[:, 0] == 0).all() and (c[:, 2] == 0).all()

    @pytest.mark.parametrize("dims", [(4, 8, 2), (5, 3, 7), (1, 9, 1, 16), (16, 16), (2, 2, 2)])
    def test_exhaustive_bijection(self, at, dims):
        lay = at.build_masks(dims)
        coords = np.array(list(np.ndindex(*dims)), dtype=np.int64)
        words = at.linearize_array(lay, coords)
        assert np.array_equal(at.delinearize_array(lay, words), coords)
        assert len(np.unique(words[:, 0])) == math.prod(dims)
        if lay.total_bits == sum(lay.bits) and 1 << lay.total_bits == math.prod(dims):
            assert set(words[:, 0].tolist()) == set(range(1 << lay.total_bits))

    @pytest.mark.parametrize("dims", [(4, 8, 2), (5, 3, 7), (1 << 40, 3, 1 << 40, 1 << 40),
                                      (40_000_000, 20_000_000, 1_000_000), (10_000_000, 5_000_000, 2000, 500)])
    def test_array_matches_oracle(self, at, dims):
        rng = np.random.default_rng(7)
        lay = at.build_masks(dims)
        coords = rng.integers(0, dims, size=(5000, len(dims)), dtype=np.int64)
        words = at.linearize_array(lay, coords)
        assert words.dtype == np.uint64 and words.shape == (5000, lay.n_words)
        olay = orc.build_layout(dims)
        assert np.array_equal(words, orc.encode(olay, coords))
        assert np.array_equal(at.delinearize_array(lay, words), coords)
        for n in range(len(dims)):
            assert np.array_equal(at.extract_mode_array(lay, words, n), coords[:, n])
        # scalar path agrees for a few rows (128-bit combine, layout.py:105-116)
        for row, w in zip(coords[:5], words[:5]):
            assert at.linearize(lay, row) == sum(int(x) << (64 * i) for i, x in enumerate(w))

    def test_bad_word_shape(self, at):
        lay = at.build_masks((4, 8, 2))
        with pytest.raises(ValueError):
            at.delinearize_array(lay, np.zeros((3, 2), dtype=np.uint64))

    def test_large_round_trip(self, at):
        """Size-independent property at 20M elements: decode(encode(x)) == x."""
        import torch

        rng = np.random.default_rng(3)
        dims = (200_000, 150_000, 100_000)
        lay = at.build_masks(dims)
        coords = torch.from_numpy(rng.integers(0, dims, size=(20_000_000, 3), dtype=np.int64)).cuda()
        keys = at.linearize_array(lay, coords)
        back = at.delinearize_array(lay, keys)
        assert torch.equal(back, coords)
