"""Host-side logic of the drop-in (no GPU): layout rule, partition offsets,
conflict-plan sweep, argument validation, generator.  Checked against the
oracle and the reference-produced golden fixtures."""

import types

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden
from oracle import alto_oracle as orc
from paper_2102_10245_b200 import synth
from paper_2102_10245_b200.format import (ConflictPlan, PartitionSet, Strategy, partition_offsets, plan_conflicts,
                                          shared_ranges)
from paper_2102_10245_b200.layout import WidthOverflowError, bits_for, build_masks


class TestBuildMasks:
    """pkg/tests/test_layout.py:28-73 goldens."""

    def test_worked_example_masks(self):
        lay = build_masks((4, 8, 2))
        assert lay.bits == (2, 3, 1) and lay.total_bits == 6 and lay.width == 64
        assert lay.masks == (0b001010, 0b110100, 0b000001)

    def test_all_singleton(self):
        lay = build_masks((1, 1, 1))
        assert lay.total_bits == 0 and lay.masks == (0, 0, 0)

    def test_group_order(self):
        lay = build_masks((5, 3, 7))
        assert lay.bits == (3, 2, 3)
        assert lay.positions == ((1, 4, 6), (0, 3), (2, 5, 7))
        assert lay.masks == (0x52, 0x09, 0xA4)

    def test_tie_break(self):
        assert build_masks((4, 4)).positions == ((0, 2), (1, 3))

    def test_ascending_slots(self):
        for slots in build_masks((100, 3, 1000, 17)).positions:
            assert list(slots) == sorted(slots)

    def test_width(self):
        assert build_masks((1 << 32, 1 << 32)).width == 64
        assert build_masks((1 << 33, 1 << 32)).width == 128
        assert build_masks((1 << 43, 1 << 43, 1 << 42)).width == 128
        with pytest.raises(WidthOverflowError):
            build_masks((1 << 43, 1 << 43, 1 << 43))
        with pytest.raises(ValueError):
            build_masks((4, 0, 2))

    def test_bits_for(self):
        assert [bits_for(d) for d in (1, 2, 3, 4, 5, 8, 9)] == [0, 1, 2, 2, 3, 3, 4]

    @pytest.mark.parametrize("name", GOLDEN_CASES)
    def test_golden_layouts(self, name):
        _, meta = load_golden(name)
        lay = build_masks(meta["dims"])
        assert [list(p) for p in lay.positions] == meta["positions"]
        assert [str(m) for m in lay.masks] == meta["masks"]
        assert (lay.total_bits, lay.width) == (meta["total_bits"], meta["width"])

    def test_random_shapes_match_oracle(self):
        rng = np.random.default_rng(0)
        for _ in range(300):
            n = int(rng.integers(1, 7))
            dims = tuple(int(d) for d in rng.integers(1, 1 << 20, size=n))
            a, b = build_masks(dims), orc.build_layout(dims)
            assert a.positions == b.positions and a.masks == b.masks and a.width == b.width


class TestPartitionOffsets:
    @pytest.mark.parametrize("m,count", [(6, 2), (500, 7), (10, 10), (0, 1), (1, 1), (1000003, 148)])
    def test_balanced_larger_first(self, m, count):
        offs = partition_offsets(m, count)
        assert offs.tolist() == orc.offsets_for(m, count).tolist()
        sizes = np.diff(offs)
        assert sizes.max() - sizes.min() <= 1 and sorted(sizes, reverse=True) == list(sizes)


def _fake_tensor(dims, nnz):
    return types.SimpleNamespace(layout=build_masks(dims), nnz=nnz)


class TestPlanConflicts:
    @pytest.mark.parametrize("name", GOLDEN_CASES)
    def test_golden_plans(self, name):
        data, meta = load_golden(name)
        t = _fake_tensor(meta["dims"], meta["nnz"])
        for count in meta["counts"]:
            parts = PartitionSet(data[f"L{count}_offsets"], data[f"L{count}_intervals"], ())
            for mode in range(len(meta["dims"])):
                for force in ("auto", "atomic", "buffered"):
                    plan = plan_conflicts(t, parts, mode, None if force == "auto" else Strategy(force))
                    want = meta["plans"][f"L{count}_m{mode}_{force}"]
                    assert plan.strategy.value == want["strategy"]
                    assert plan.reuse == want["reuse"]
                    assert plan.flag_bit == want["flag_bit"]
                    got = None if plan.overlaps is None else [[list(r) for r in o] for o in plan.overlaps]
                    assert got == want["overlaps"]
                    assert plan.offsets is parts.offsets

    def test_sweep_equals_pairwise_scan(self):
        """The coverage sweep reproduces format.py:234-246 on random intervals,
        including empty partitions, duplicates, nesting and adjacency."""
        rng = np.random.default_rng(7)
        for trial in range(400):
            L = int(rng.integers(1, 12))
            lo = rng.integers(0, 40, size=L)
            hi = lo + rng.integers(-1, 15, size=L)
            empty = rng.random(L) < 0.1
            lo[empty], hi[empty] = 0, -1
            iv = np.stack([lo, hi], axis=1)
            ref = orc.plan(orc.build_layout((64, 4)), 100, iv[:, None, :].repeat(2, axis=1), 0, "atomic")
            assert shared_ranges(iv) == ref["overlaps"], (iv.tolist(), trial)

    def test_mode_range(self):
        t = _fake_tensor((4, 8, 2), 6)
        parts = PartitionSet(np.array([0, 3, 6]), np.zeros((2, 3, 2), np.int64), ())
        with pytest.raises(ValueError):
            plan_conflicts(t, parts, 3)

    def test_reuse_threshold(self):
        t = _fake_tensor((10, 50, 2), 100)
        parts = PartitionSet(np.array([0, 100]), np.array([[[0, 9], [0, 49], [0, 1]]]), ())
        assert plan_conflicts(t, parts, 0).strategy is Strategy.BUFFERED
        assert plan_conflicts(t, parts, 1).strategy is Strategy.ATOMIC
        assert plan_conflicts(t, parts, 0).reuse == 10.0

    def test_plan_is_frozen_and_replaceable(self):
        import dataclasses

        plan = ConflictPlan(0, Strategy.ATOMIC, 1.0, np.array([0, 1]), ((),), 6)
        assert dataclasses.replace(plan, flag_bit=None).flag_bit is None
        with pytest.raises(dataclasses.FrozenInstanceError):
            plan.mode = 1


class TestSynth:
    def test_distinct_and_seeded(self):
        a = synth.make_tensor(2, nnz=20_000)
        b = synth.make_tensor(2, nnz=20_000)
        assert np.array_equal(a.coords, b.coords) and np.array_equal(a.values, b.values)
        packed = a.coords[:, 0] * (1 << 40) + a.coords[:, 1] * (1 << 20) + a.coords[:, 2]
        assert np.unique(packed).size == 20_000
        assert a.values.dtype == np.float32
        assert (a.coords < np.asarray(a.config.dims)).all() and (a.coords >= 0).all()

    def test_zipf_head_heavier(self):
        t = synth.make_tensor(2, nnz=50_000)
        c = t.coords[:, 0]
        assert (c < 100).mean() > 0.3  # bounded Zipf(1.1) puts ~half the mass below 100

    def test_wide_config_packs_two_columns(self):
        t = synth.make_tensor(5, nnz=5_000)
        assert t.coords.shape == (5_000, 3)
        assert len(np.unique(t.coords, axis=0)) == 5_000


class TestModeStreamPairs:
    """ms_pairs: which input modes the mode-stream kernel gathers as one
    product-table row (smallest two, then the next two, within the byte cap)."""

    def test_cfg4_pairs(self):
        import importlib

        mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
        dims = synth.CONFIGS[4].dims  # 1000 x 1000 x 1000 x 100 x 50
        assert mk.ms_pairs(dims, 0, 16, 4, 64 << 20) == [(4, 3), (1, 2)]
        assert mk.ms_pairs(dims, 3, 16, 4, 64 << 20) == [(4, 0), (1, 2)]
        assert mk.ms_pairs(dims, 0, 16, 4, 1 << 20) == [(4, 3)]  # 5000 rows x 64 B fit, 1M rows do not

    def test_not_paired(self):
        import importlib

        mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
        assert mk.ms_pairs(synth.CONFIGS[2].dims, 0, 16, 4, 64 << 20) == []  # order 3
        assert mk.ms_pairs(synth.CONFIGS[4].dims, 0, 32, 4, 64 << 20) == []  # rank 32
        assert mk.ms_pairs(synth.CONFIGS[4].dims, 0, 16, 8, 64 << 20) == []  # float64
        assert mk.ms_pairs(synth.CONFIGS[4].dims, 0, 16, 4, 0) == []  # disabled
        assert mk.ms_pairs(synth.CONFIGS[3].dims, 0, 16, 4, 64 << 20) == [(3, 2)]  # 2000 x 500 x 64 B = 64e6 B
        assert mk.ms_pairs(synth.CONFIGS[3].dims, 0, 16, 4, 64_000_000 - 1) == []


class TestBenchContract:
    """bench.py's reference arm (CPU only) prints one JSON line with the
    contract's keys; the argument parser accepts every documented flag."""

    def test_reference_arm_runs(self):
        import json
        import subprocess
        import sys

        from conftest import ROOT

        out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
                              "--cpu-sample", "20000"], cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        line = json.loads(out.stdout.strip().splitlines()[-1])
        for k in ("metric", "value", "unit", "impl", "cpu_baseline", "e2e", "config"):
            assert k in line
        assert line["impl"] == "reference" and line["value"] > 0

    def test_flags_parse(self):
        import subprocess
        import sys

        from conftest import ROOT

        out = subprocess.run([sys.executable, "bench.py", "--help"], cwd=ROOT, capture_output=True, text=True,
                             timeout=120)
        assert out.returncode == 0
        for flag in ("--gpus", "--steps", "--warmup", "--impl", "--config", "--skip-cpu", "--skip-cpals", "--out"):
            assert flag in out.stdout
