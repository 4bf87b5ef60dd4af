"""Device ALTO build / sort / partition / flags: bit-exact against the
reference-produced golden fixtures and the oracle."""

import dataclasses
import hashlib

import numpy as np
import pytest

from conftest import EXAMPLE_LINEAR, GOLDEN_CASES, load_golden
from oracle import alto_oracle as orc
from paper_2102_10245_b200 import synth

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden_inputs(data, meta):
    if "coords" in data:
        return data["coords"], data["values"]
    st = synth.make_tensor(1) if meta["name"] == "cfg1" else synth.make_tensor(2, nnz=200_000)
    return st.coords, st.values.astype(np.float64)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_build_partition_plan_flags_match_reference(at, name):
    data, meta = load_golden(name)
    coords, values = golden_inputs(data, meta)
    alto = at.build_alto(at.CooTensor(meta["dims"], coords, values))
    assert sha(alto.indices) == meta["indices_sha"]
    assert sha(alto.values) == meta["sorted_values_sha"]
    for count in meta["counts"]:
        parts = at.partition(alto, count)
        assert np.array_equal(parts.offsets, data[f"L{count}_offsets"])
        assert np.array_equal(parts.intervals, data[f"L{count}_intervals"])
        assert [[str(a), str(b)] for a, b in parts.spans] == meta[f"L{count}_spans"]
        for mode in range(len(meta["dims"])):
            plan = at.plan_conflicts(alto, parts, mode, force_strategy=at.Strategy.ATOMIC)
            key = f"L{count}_m{mode}_atomic"
            if plan.flag_bit is not None:
                flagged = at.apply_boundary_flags(alto, plan)
                assert sha(flagged.indices) == meta[key + "_flagged_sha"]
                assert np.array_equal(at.read_flags(flagged, plan.flag_bit),
                                      orc.read_flags(flagged.indices, plan.flag_bit))
                assert np.array_equal(at.clear_flags(flagged, plan.flag_bit).indices, alto.indices)


class TestBuildAlto:
    def test_sorted_positions(self, example_alto):
        assert example_alto.linear_positions() == EXAMPLE_LINEAR
        assert example_alto.values[-1] == 6.0

    def test_round_trip(self, at, example_coo, example_alto):
        assert example_alto.to_coo().isequal(example_coo)
        t = at.random_tensor((60, 50, 40), 10000, seed=2)
        back = at.build_alto(t).to_coo()
        assert np.array_equal(back.coords, t.coords) and np.array_equal(back.values, t.values)

    def test_single_element_and_empty(self, at):
        assert at.build_alto(at.CooTensor((4, 4), [[0, 0]], [1.0])).linear_positions() == [0]
        e = at.build_alto(at.CooTensor((4, 8, 2), np.empty((0, 3), np.int64), np.empty(0)))
        assert e.nnz == 0 and e.indices.shape == (0, 1)

    def test_duplicates_rejected(self, at):
        with pytest.raises(ValueError, match="coalesce"):
            at.build_alto(at.CooTensor((4, 4), [[1, 2], [1, 2]], [1.0, 2.0]))
        wide = (1 << 40, 1 << 40)
        with pytest.raises(ValueError, match="coalesce"):
            at.build_alto(at.CooTensor(wide, [[5, 1 << 39], [3, 3], [5, 1 << 39]], [1.0, 2.0, 3.0]))

    def test_layout_dims_must_match(self, at):
        with pytest.raises(ValueError, match="dims"):
            at.build_alto(at.CooTensor((4, 4), [[0, 0]], [1.0]), layout=at.build_masks((4, 8)))

    def test_wide_round_trip(self, at):
        rng = np.random.default_rng(9)
        dims = (1 << 40, 1 << 30, 1 << 40)
        c = np.unique(rng.integers(0, dims, size=(300, 3), dtype=np.int64), axis=0)
        t = at.CooTensor(dims, c, rng.random(len(c)))
        alto = at.build_alto(t)
        assert alto.layout.width == 128 and alto.indices.shape[1] == 2
        assert alto.to_coo().isequal(t)

    def test_float32_storage(self, at):
        st = synth.make_tensor(2, nnz=50_000)
        coo = at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64))
        a64 = at.build_alto(coo)
        a32 = at.build_alto(coo, dtype="float32")
        assert np.array_equal(a64.indices, a32.indices)
        assert np.array_equal(a64.values, a32.values)  # fp32-rounded inputs upcast exactly


class TestPartition:
    @pytest.mark.parametrize("count", [1, 2, 3, 5, 7])
    def test_balance(self, at, count):
        alto = at.build_alto(at.random_tensor((20, 30, 10), 500, seed=4))
        parts = at.partition(alto, count)
        sizes = np.diff(parts.offsets)
        assert sizes.max() - sizes.min() <= 1 and sorted(sizes, reverse=True) == list(sizes)

    def test_tight_sound_and_singletons(self, at):
        alto = at.build_alto(at.random_tensor((11, 13, 9, 8), 700, seed=21))
        coords = orc.decode(orc.build_layout(alto.dims), alto.indices)
        for count in (1, 2, 3, 7, alto.nnz):
            parts = at.partition(alto, count)
            for l in range(count):
                seg = coords[parts.offsets[l]:parts.offsets[l + 1]]
                assert (seg.min(0) == parts.intervals[l, :, 0]).all()
                assert (seg.max(0) == parts.intervals[l, :, 1]).all()
            for (a0, a1), (b0, b1) in zip(parts.spans, parts.spans[1:]):
                assert a0 <= a1 < b0 <= b1

    def test_count_range(self, at, example_alto):
        with pytest.raises(ValueError):
            at.partition(example_alto, 0)
        with pytest.raises(ValueError):
            at.partition(example_alto, example_alto.nnz + 1)


class TestFlags:
    def test_worked_example(self, at, example_alto):
        parts = at.partition(example_alto, 2)
        plan = at.plan_conflicts(example_alto, parts, 0)
        assert plan.overlaps == (((1, 3),), ((1, 3),)) and plan.flag_bit == 6
        flagged = at.apply_boundary_flags(example_alto, plan)
        assert at.read_flags(flagged, 6).tolist() == [True, True, False, True, True, True]
        assert at.clear_flags(flagged, 6).linear_positions() == EXAMPLE_LINEAR

    def test_single_partition_flags_nothing(self, at, example_alto):
        plan = at.plan_conflicts(example_alto, at.partition(example_alto, 1), 0)
        assert not at.read_flags(at.apply_boundary_flags(example_alto, plan), plan.flag_bit).any()

    def test_coverage_of_shared_rows(self, at):
        alto = at.build_alto(at.random_tensor((12, 10, 8), 400, seed=6))
        parts = at.partition(alto, 5)
        coords = at.delinearize_array(alto.layout, alto.indices)
        for mode in range(3):
            plan = at.plan_conflicts(alto, parts, mode, force_strategy=at.Strategy.ATOMIC)
            flags = at.read_flags(at.apply_boundary_flags(alto, plan), plan.flag_bit)
            writers = {}
            for l in range(parts.count):
                for c in np.unique(coords[parts.offsets[l]:parts.offsets[l + 1], mode]):
                    writers.setdefault(int(c), set()).add(l)
            shared = {c for c, w in writers.items() if len(w) > 1}
            assert all(flags[i] for i in range(alto.nnz) if int(coords[i, mode]) in shared)

    def test_arbitrary_offsets(self, at):
        """Plans whose offsets are not the equal-size split (including empty
        partitions) are flagged exactly as the reference does
        (format.py:274-284 loops over plan.offsets)."""
        alto = at.build_alto(at.random_tensor((30, 20, 16), 2000, seed=9))
        lay = orc.build_layout(alto.layout.dims)
        words = alto.indices
        m = alto.nnz
        offs = np.array([0, 5, 5, 400, 1111, m - 3, m], dtype=np.int64)
        for mode in range(3):
            base = at.plan_conflicts(alto, at.partition(alto, len(offs) - 1), mode,
                                     force_strategy=at.Strategy.ATOMIC)
            coords = orc.decode(lay, words, mode)
            ovl = []
            for l in range(len(offs) - 1):
                mine = set(coords[offs[l]:offs[l + 1]].tolist())
                other = set(coords[:offs[l]].tolist()) | set(coords[offs[l + 1]:].tolist())
                rows = sorted(mine & other)
                ovl.append(tuple((r, r) for r in rows))
            plan = dataclasses.replace(base, offsets=offs, overlaps=tuple(ovl))
            got = at.apply_boundary_flags(alto, plan).indices
            want = orc.flag(lay, words, offs, mode, plan.overlaps, plan.flag_bit)
            assert np.array_equal(got, want), mode

    def test_rejections(self, at, example_alto):
        parts = at.partition(example_alto, 2)
        buf = at.plan_conflicts(example_alto, parts, 0, force_strategy=at.Strategy.BUFFERED)
        with pytest.raises(ValueError, match="atomic"):
            at.apply_boundary_flags(example_alto, buf)
        plan = at.plan_conflicts(example_alto, parts, 0)
        with pytest.raises(ValueError, match="unused"):
            at.apply_boundary_flags(example_alto, dataclasses.replace(plan, flag_bit=None))
        other = at.build_alto(at.random_tensor((4, 8, 2), 3, seed=0))
        with pytest.raises(ValueError, match="match"):
            at.apply_boundary_flags(other, plan)


class TestScale:
    def test_cfg2_law_2m_sorted_unique_and_matches_oracle_order(self, at):
        """2M-element build on the cfg2 law: keys strictly ascending (sortedness +
        no duplicates), multiset of keys equals the oracle's encoding, and
        values co-permuted (checksum)."""
        st = synth.make_tensor(2, nnz=2_000_000)
        coo = at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64))
        alto = at.build_alto(coo, dtype="float32")
        k = alto.indices[:, 0]
        assert (k[1:] > k[:-1]).all()
        olay = orc.build_layout(st.config.dims)
        words, vals = orc.build(olay, st.coords, st.values.astype(np.float64))
        assert np.array_equal(alto.indices, words)
        assert np.array_equal(alto.values, vals)
