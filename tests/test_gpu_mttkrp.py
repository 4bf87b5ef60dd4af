"""Device MTTKRP engines against the reference-produced fixtures and the
oracle.  The exact-order engine must be BITWISE equal to the reference
(mttkrp_seq, Buffered mttkrp_par) on float64 data; the streaming kernel
within 1e-12 (fp64) / 1e-5 (fp32) relative Frobenius error."""

import dataclasses

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden, rel_error
from oracle import alto_oracle as orc
from paper_2102_10245_b200 import synth

pytestmark = pytest.mark.gpu


def seeded_factors(dims, rank, seed=0):
    rng = np.random.default_rng(seed)
    return [rng.random((d, rank)) for d in dims]


def golden_setup(at, name):
    data, meta = load_golden(name)
    if "coords" in data:
        coords, values = data["coords"], data["values"]
    else:
        st = synth.make_tensor(1) if name == "cfg1" else synth.make_tensor(2, nnz=200_000)
        coords, values = st.coords, st.values.astype(np.float64)
    coo = at.CooTensor(meta["dims"], coords, values)
    rng = np.random.default_rng(meta["fseed"])
    factors = [rng.random((d, meta["rank"])) for d in meta["dims"]]
    return data, meta, coo, factors


def compare(data, meta, key, out, tol):
    if meta.get("project"):
        u = np.random.default_rng(99).random(meta["rank"])
        assert rel_error(out @ u, data[key + "_proj"]) <= max(tol, 1e-15), key
        return
    if tol == 0:
        assert np.array_equal(out, data[key]), (key, rel_error(out, data[key]))
    else:
        assert rel_error(out, data[key]) <= tol, (key, rel_error(out, data[key]))


MTTKRP_CASES = [n for n in GOLDEN_CASES if load_golden(n)[1]["with_mttkrp"]]


@pytest.mark.parametrize("name", MTTKRP_CASES)
def test_engines_match_reference(at, name):
    data, meta, coo, factors = golden_setup(at, name)
    alto = at.build_alto(coo)
    for mode in range(len(meta["dims"])):
        # exact-order engine == reference mttkrp_seq, bit for bit
        compare(data, meta, f"m{mode}_seq", at.mttkrp_seq(alto, factors, mode), 0)
        compare(data, meta, f"m{mode}_oracle", at.mttkrp_oracle(coo, factors, mode), 0)
        for count in meta["counts"]:
            parts = at.partition(alto, count)
            plan = at.plan_conflicts(alto, parts, mode, force_strategy=at.Strategy.BUFFERED)
            compare(data, meta, f"L{count}_m{mode}_buffered_mttkrp",
                    at.mttkrp_par(alto, parts, plan, factors, mode, workers=4), 0)
            plan = at.plan_conflicts(alto, parts, mode, force_strategy=at.Strategy.ATOMIC)
            run = at.apply_boundary_flags(alto, plan) if plan.flag_bit is not None else alto
            compare(data, meta, f"L{count}_m{mode}_atomic_mttkrp",
                    at.mttkrp_par(run, parts, plan, factors, mode, workers=4), 1e-12)


class TestParallelSemantics:
    """pkg/tests/test_mttkrp.py:117-226 on the device."""

    @pytest.fixture
    def setup(self, at):
        t = at.random_tensor((25, 30, 18), 2500, seed=10)
        return t, at.build_alto(t), seeded_factors(t.dims, 8, seed=11)

    def test_buffered_bitwise_deterministic(self, at, setup):
        _, alto, factors = setup
        runs = [at.mttkrp(alto, factors, 1, workers=w, partitions=6, strategy=at.Strategy.BUFFERED)
                for w in (1, 2, 4, 8)]
        for out in runs[1:]:
            assert np.array_equal(runs[0], out)

    def test_strategy_equivalence(self, at, setup):
        t, alto, factors = setup
        for mode in range(3):
            ref = orc.mttkrp_coo(t.coords, t.values, factors, mode)
            outs = [at.mttkrp_seq(alto, factors, mode)]
            for s in at.Strategy:
                outs.append(at.mttkrp(alto, factors, mode, workers=4, partitions=8, strategy=s))
            for a in outs:
                assert rel_error(a, ref) <= 1e-12

    def test_flag_soundness(self, at, setup):
        _, alto, factors = setup
        parts = at.partition(alto, 8)
        for mode in range(3):
            plan = at.plan_conflicts(alto, parts, mode, force_strategy=at.Strategy.ATOMIC)
            out = at.mttkrp_par(at.apply_boundary_flags(alto, plan), parts, plan, factors, mode, workers=4)
            all_out = at.mttkrp_par(alto, parts, dataclasses.replace(plan, flag_bit=None), factors, mode, 4)
            assert rel_error(out, all_out) <= 1e-12

    def test_linearity(self, at, setup):
        _, alto, factors = setup
        scaled = at.AltoTensor(alto.layout, alto.indices, 3.5 * alto.values)
        for s in at.Strategy:
            a = at.mttkrp(scaled, factors, 2, workers=2, partitions=4, strategy=s)
            b = 3.5 * at.mttkrp(alto, factors, 2, workers=2, partitions=4, strategy=s)
            assert rel_error(a, b) <= 1e-12

    def test_atomic_requires_flags(self, at, setup):
        _, alto, factors = setup
        parts = at.partition(alto, 8)
        plan = at.plan_conflicts(alto, parts, 0, force_strategy=at.Strategy.ATOMIC)
        assert any(plan.overlaps)
        with pytest.raises(ValueError, match="flags"):
            at.mttkrp_par(alto, parts, plan, factors, 0, workers=2)
        # the guard's answer is cached per tensor: still raises on repeat,
        # and a flagged tensor passes it on every call
        with pytest.raises(ValueError, match="flags"):
            at.mttkrp_par(alto, parts, plan, factors, 0, workers=2)
        flagged = at.apply_boundary_flags(alto, plan)
        a = at.mttkrp_par(flagged, parts, plan, factors, 0, workers=2)
        b = at.mttkrp_par(flagged, parts, plan, factors, 0, workers=2)
        assert ("anyflag", plan.flag_bit) in flagged._cache
        assert rel_error(a, b) <= 1e-12

    def test_plan_mismatch(self, at, setup):
        _, alto, factors = setup
        parts, other = at.partition(alto, 4), at.partition(alto, 5)
        plan = at.plan_conflicts(alto, parts, 0)
        with pytest.raises(ValueError, match="mode"):
            at.mttkrp_par(alto, parts, plan, factors, 1, workers=1)
        with pytest.raises(ValueError, match="partition"):
            at.mttkrp_par(alto, other, plan, factors, 0, workers=1)
        with pytest.raises(ValueError, match="workers"):
            at.mttkrp_par(alto, parts, plan, factors, 0, workers=0)

    def test_shape_validation(self, at):
        t = at.random_tensor((4, 4, 4), 10, seed=0)
        good = seeded_factors(t.dims, 2)
        with pytest.raises(ValueError, match="mode"):
            at.mttkrp_oracle(t, good, 3)
        with pytest.raises(ValueError, match="factor matrices"):
            at.mttkrp_oracle(t, good[:2], 0)
        with pytest.raises(ValueError, match="rows"):
            at.mttkrp_oracle(t, [np.ones((5, 2)), np.ones((4, 2)), np.ones((4, 2))], 0)
        with pytest.raises(ValueError, match="rank"):
            at.mttkrp_oracle(t, [np.ones((4, 2)), np.ones((4, 3)), np.ones((4, 2))], 0)

    def test_empty_tensor(self, at):
        e = at.AltoTensor(at.build_masks((4, 8, 2)), np.empty((0, 1), np.uint64), np.empty(0))
        assert not at.mttkrp_seq(e, seeded_factors((4, 8, 2), 3), 1).any()
        out = at.mttkrp(e, seeded_factors((4, 8, 2), 2), 0, workers=4)
        assert out.shape == (4, 2) and not out.any()

    def test_pipeline_clamping(self, at):
        t = at.random_tensor((4, 100, 4), 64, seed=14)
        alto = at.build_alto(t)
        factors = seeded_factors(t.dims, 2, seed=15)
        assert rel_error(at.mttkrp(alto, factors, 1, workers=2, partitions=1000),
                         orc.mttkrp_coo(t.coords, t.values, factors, 1)) <= 1e-12

    def test_order_one_and_two(self, at):
        t1 = at.CooTensor((10,), [[1], [4], [7]], [1.0, 2.0, 3.0])
        a1 = at.build_alto(t1)
        f = seeded_factors((10,), 3)
        assert np.array_equal(at.mttkrp_seq(a1, f, 0), orc.mttkrp_seq(orc.build_layout((10,)), a1.indices,
                                                                       a1.values, f, 0))
        t2 = at.random_tensor((30, 20), 200, seed=1)
        a2 = at.build_alto(t2)
        f2 = seeded_factors((30, 20), 4)
        for mode in range(2):
            ref = orc.mttkrp_coo(t2.coords, t2.values, f2, mode)
            assert rel_error(at.mttkrp(a2, f2, mode, partitions=3, strategy=at.Strategy.ATOMIC), ref) <= 1e-12


class TestStreamKernel:
    """The fast path at fp32 against the fp64 oracle (north-star bar 1e-5)."""

    WIDE = synth.SynthConfig("cfg9", (1 << 22, 1 << 22, 1 << 21), 0, (("zipf", 1.05),) * 3, "uniform01",
                             "float32", 16)

    @pytest.mark.parametrize("cfg,nnz,rank", [(2, 300_000, 16), (3, 200_000, 32), (4, 300_000, 16),
                                              ("wide", 300_000, 16), (1, 100_000, 16)])
    def test_configs_vs_oracle(self, at, cfg, nnz, rank):
        """fp32 configs at 1e-5 (cfg1: fp64 at 1e-12).  'wide' = 65-bit,
        128-bit-key layout with the cfg5 Zipf law at materialisable extents."""
        import torch

        from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_stream

        st = synth.make_tensor(self.WIDE if cfg == "wide" else cfg, nnz=nnz)
        if cfg == "wide":
            cfg = 9
        dims = st.config.dims
        coo = at.CooTensor(dims, st.coords, st.values.astype(np.float64))
        fp32 = st.config.value_dtype == "float32"
        alto = at.build_alto(coo, dtype="float32" if fp32 else "float64")
        rng = np.random.default_rng(synth.SEED_FACTOR_BASE + cfg)
        factors = [rng.random((d, rank)).astype(np.float32 if fp32 else np.float64) for d in dims]
        fdev = factors_to_device(factors)
        f64 = [f.astype(np.float64) for f in factors]
        tol = 1e-5 if fp32 else 1e-12
        for mode in range(len(dims)):
            ref = orc.mttkrp_coo(st.coords, st.values.astype(np.float64), f64, mode)
            for tile in (256, 512, 1024):
                out = mttkrp_stream(alto, fdev, mode, tile=tile).cpu().numpy()
                assert rel_error(out, ref) <= tol, (cfg, mode, tile, rel_error(out, ref))
            torch.cuda.synchronize()

    @pytest.mark.parametrize("cfg,nnz,rank", [(2, 400_000, 16), (3, 150_000, 32), (4, 300_000, 16),
                                              (3, 150_000, 16), (5, 200_000, 32), (4, 200_000, 32)])
    def test_float32_output(self, at, cfg, nnz, rank):
        """float32 output (RED.F32x4 merge, hot rows in float64) vs the fp64 oracle at 1e-5.
        The (cfg, rank) pairs cover the cooperative kernel (order 3, rank 16), the blocked
        kernel at rank 32 (orders 3-5, one-word delta keys on the 128-bit layouts of cfg3 /
        cfg5, two-word keys on cfg3's short modes) and with paired input modes (cfg4 and
        cfg3 at rank 16: pairs + delta keys)."""
        import torch

        from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_stream

        st = synth.make_tensor(cfg, nnz=nnz)
        dims = st.config.dims
        alto = at.build_alto(at.CooTensor(dims, st.coords, st.values.astype(np.float64)), dtype="float32")
        rng = np.random.default_rng(7)
        factors = [rng.random((d, rank)).astype(np.float32) for d in dims]
        fdev = factors_to_device(factors)
        for mode in range(len(dims)):
            ref = orc.mttkrp_coo(st.coords, st.values.astype(np.float64), [f.astype(np.float64) for f in factors],
                                 mode)
            out = mttkrp_stream(alto, fdev, mode, out_dtype=torch.float32)
            assert out.dtype == torch.float32
            assert rel_error(out.double().cpu().numpy(), ref) <= 1e-5
            nohot = mttkrp_stream(alto, fdev, mode, out_dtype=torch.float32, hot=False)
            assert rel_error(nohot.double().cpu().numpy(), ref) <= 1e-5

    @pytest.mark.parametrize("cfg", [2, "wide"])
    def test_stream_plan(self, at, cfg):
        """Per-tensor packed keys and per-mode sub-tile order (alto_pack_keys /
        alto_subtile_order): fields decode to the coordinates; pos is, per
        128-element sub-tile, the stable row-sorted slot; planned == unplanned."""
        import torch

        from paper_2102_10245_b200.mttkrp import (factors_to_device, mttkrp_stream, packed_keys,
                                                  subtile_order)

        st = synth.make_tensor(self.WIDE if cfg == "wide" else cfg, nnz=100_003)
        dims = st.config.dims
        alto = at.build_alto(at.CooTensor(dims, st.coords, st.values.astype(np.float64)), dtype="float32")
        lay = alto.layout
        coords = orc.decode(orc.build_layout(dims), alto.indices)
        pk = packed_keys(alto).cpu().numpy().view(np.uint64)
        ints = [sum(int(w) << (64 * i) for i, w in enumerate(row)) for row in pk[:2000]]
        off = 0
        for n in range(len(dims)):
            got = np.array([(v >> off) & ((1 << lay.bits[n]) - 1) for v in ints])
            assert np.array_equal(got, coords[:2000, n])
            off += lay.bits[n]
        for mode in range(len(dims)):
            pos = subtile_order(alto, mode).cpu().numpy()[:alto.nnz].astype(np.int64)
            for s0 in range(0, alto.nnz, 128 * 97):
                seg = slice(s0, min(s0 + 128, alto.nnz))
                p, r = pos[seg], coords[seg, mode]
                assert sorted(p.tolist()) == list(range(len(p)))
                if r.max() - r.min() < 512:
                    order = np.argsort(p)
                    assert (np.diff(r[order]) >= 0).all()
                    assert np.array_equal(order, np.argsort(r, kind="stable"))
        rng = np.random.default_rng(4)
        fdev = factors_to_device([rng.random((d, 16)).astype(np.float32) for d in dims])
        for mode in range(len(dims)):
            b = mttkrp_stream(alto, fdev, mode, out_dtype=torch.float32, planned=False).double().cpu().numpy()
            for variant in (True, "pos"):
                a = mttkrp_stream(alto, fdev, mode, out_dtype=torch.float32, planned=variant).double().cpu().numpy()
                assert rel_error(a, b) <= 1e-6, variant

    @pytest.mark.parametrize("rrobin", [0, 1, 3])
    @pytest.mark.parametrize("order", [0, 1])
    @pytest.mark.parametrize("cfg", [2, "wide", 4])
    def test_mode_stream_layout(self, at, monkeypatch, cfg, order, rrobin):
        """Per-mode stream (alto_mode_stream): the ALTO stream stably sorted by
        the mode's coordinate — as a whole (order 1, ALTO_MS_ROW_MAJOR) or tile
        by tile (order 0) — cut into tiles of T stored as 8 interleaved slices;
        keys re-pack the coordinates (input modes ascending, then the mode; no
        field straddles a 64-bit word) with the hot flag on the top bit."""
        import importlib

        import torch

        mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
        monkeypatch.setattr(mk, "MS_ORDER", order)
        monkeypatch.setattr(mk, "MS_RR", rrobin)
        st = synth.make_tensor(self.WIDE if cfg == "wide" else cfg, nnz=60_001)
        dims = st.config.dims
        alto = at.build_alto(at.CooTensor(dims, st.coords, st.values.astype(np.float64)), dtype="float32")
        lay = alto.layout
        W = lay.n_words
        coords = orc.decode(orc.build_layout(dims), alto.indices)
        vals = alto.vals.cpu().numpy()
        T = mk.ms_tile(alto)
        assert T == 128  # small tensor: shortest tiles
        for mode in range(len(dims)):
            ms = mk.mode_stream(alto, mode)
            assert ms is not None
            sk, sv, tile, rr, base = ms
            assert tile == T
            delta = base is not None
            assert delta == (W == 2 and order == 1)  # ALTO_MS_DELTA for 128-bit layouts, row-major streams
            KW = 1 if delta else W
            sk = sk.cpu().numpy().view(np.uint64).reshape(-1, KW)
            sv = sv.cpu().numpy()
            if rr == 2:
                # blocked: sorted element k*gpw+s of a warp step is stored at s*u+k (group s
                # takes sorted positions s, s+gpw, ...): back to sorted order
                u, gpw = mk.ms_block(len(dims), 16, 0 if sv.dtype == np.float32 else 1, 0)
                bperm = np.arange(sk.shape[0]).reshape(-1, gpw, u).transpose(0, 2, 1).reshape(-1)
                sk, sv = sk[bperm], sv[bperm]
            forder = [n for n in range(len(dims)) if n != mode] + [mode]
            cur, fields = 0, {}
            for n in forder:
                b = lay.bits[n]
                if delta and n == mode:
                    b = min(31, 63 - cur)  # the row-increment field
                if (cur % 64) + b > 64:
                    cur = (cur + 63) // 64 * 64
                fields[n] = (cur // 64, cur % 64, b)
                cur += b
            if delta:  # rows = group base + running sum of increments
                base = base.cpu().numpy()
                inc = ((sk[:, 0] >> np.uint64(fields[mode][1])) & np.uint64((1 << fields[mode][2]) - 1)).astype(np.int64)
                nt = (alto.nnz + T - 1) // T
                gpw = 8
                if rr == 2:
                    gpw = mk.ms_block(len(dims), 16, 0 if sv.dtype == np.float32 else 1, 0)[1]
                g = inc[:nt * T].reshape(nt, T // gpw, gpw)
                rows_all = (np.cumsum(g, axis=1) + base[:nt * gpw].reshape(nt, 1, gpw)).reshape(-1)
            hs = mk.hot_slots(alto, mode)
            hot_rows = set() if hs is None else set(hs[1][:hs[2]].cpu().numpy().tolist())
            ch = T // 8
            gperm = np.argsort(coords[:, mode], kind="stable")  # row-major order of the whole stream
            for t0 in list(range(0, alto.nnz, T))[::7] + [alto.nnz - 1 - (alto.nnz - 1) % T]:
                cnt = min(T, alto.nnz - t0)
                p = np.arange(cnt)
                idx = t0 + (p if rr else (p % ch) * 8 + p // ch)
                keys = sk[idx]
                dec = np.stack([(keys[:, fields[n][0]] >> np.uint64(fields[n][1])) & np.uint64((1 << fields[n][2]) - 1)
                                for n in range(len(dims))], 1).astype(np.int64)
                if delta:
                    dec[:, mode] = rows_all[idx]
                flag = (keys[:, KW - 1] >> np.uint64(63)).astype(bool)
                if order == 1:
                    ref = gperm[t0:t0 + cnt]
                else:
                    ref = t0 + np.argsort(coords[t0:t0 + cnt, mode], kind="stable")
                assert np.array_equal(dec, coords[ref])
                assert np.array_equal(sv[idx], vals[ref])
                assert np.array_equal(flag, np.array([r in hot_rows for r in dec[:, mode]]))
        rng = np.random.default_rng(4)
        fdev = mk.factors_to_device([rng.random((d, 16)).astype(np.float32) for d in dims])
        for mode in range(len(dims)):
            b = mk.mttkrp_stream(alto, fdev, mode, planned=False).cpu().numpy()
            a = mk.mttkrp_stream(alto, fdev, mode).cpu().numpy()
            assert rel_error(a, b) <= 3e-6  # two float32 accumulation orders
            torch.cuda.synchronize()

    @pytest.mark.parametrize("cfg", [4, "four"])
    def test_paired_input_modes(self, at, monkeypatch, cfg):
        """Paired input modes (alto_krp_pair tables, one gather for two modes):
        every mode against the float64 oracle and the unpaired kernel, plus
        the product table itself against NumPy."""
        import importlib

        import torch

        mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
        four = synth.SynthConfig("cfg8", (3000, 700, 40, 90), 0, (("zipf", 1.1),) * 2 + (("uniform", 0),) * 2,
                                 "uniform01", "float32", 16)
        st = synth.make_tensor(four if cfg == "four" else cfg, nnz=120_007)
        dims = st.config.dims
        coo = at.CooTensor(dims, st.coords, st.values.astype(np.float32).astype(np.float64))
        alto = at.build_alto(coo, dtype="float32")
        rng = np.random.default_rng(5)
        f32 = [rng.random((d, 16)).astype(np.float32) for d in dims]
        fdev = mk.factors_to_device(f32)
        for mode in range(len(dims)):
            pairs = mk.ms_pairs(dims, mode, 16, 4)
            assert pairs, (dims, mode)
            ref = orc.mttkrp_coo(st.coords, coo.values, [f.astype(np.float64) for f in f32], mode)
            a = mk.mttkrp_stream(alto, fdev, mode).cpu().numpy()
            monkeypatch.setattr(mk, "MS_PAIR_BYTES", 0)
            b = mk.mttkrp_stream(alto, fdev, mode).cpu().numpy()
            monkeypatch.setattr(mk, "MS_PAIR_BYTES", 64 << 20)
            assert rel_error(a, ref) <= 1e-5
            assert rel_error(a, b) <= 1e-6
            # the ALTO-order single-copy kernel gathers the same product tables
            p = mk.mttkrp_stream(alto, fdev, mode, planned="pos").cpu().numpy()
            assert rel_error(p, ref) <= 1e-5
        pa, pb = mk.ms_pairs(dims, 0, 16, 4)[0]
        tab = torch.empty((dims[pa] * dims[pb], 16), dtype=torch.float32, device="cuda")
        from paper_2102_10245_b200 import _lib
        _lib.check(_lib.load().alto_krp_pair(fdev[pa].data_ptr(), dims[pa], fdev[pb].data_ptr(), dims[pb], 16,
                                             _lib.ALTO_F32, tab.data_ptr(), _lib.stream_ptr()), "alto_krp_pair")
        want = (f32[pa][:, None, :] * f32[pb][None, :, :]).reshape(-1, 16)
        assert np.array_equal(tab.cpu().numpy(), want)

    @pytest.mark.parametrize("cfg,nnz", [(2, 300_001), ("wide", 70_001), (4, 1_000)])
    def test_row_counts_equal_row_index(self, at, cfg, nnz):
        """alto_row_counts (histogram) + prefix sum == the row offsets of alto_row_index (sort)."""
        import importlib

        import torch

        mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
        st = synth.make_tensor(self.WIDE if cfg == "wide" else cfg, nnz=nnz)
        dims = st.config.dims
        alto = at.build_alto(at.CooTensor(dims, st.coords, st.values.astype(np.float64)), dtype="float32")
        for mode in range(len(dims)):
            ptr = mk.row_ptr(alto, mode)  # histogram path (no row index cached yet)
            assert ("row_ptr", mode) in alto._cache
            ref = mk.row_index(alto, mode)[1]
            assert torch.equal(ptr, ref)
            want = np.concatenate([[0], np.cumsum(np.bincount(st.coords[:, mode], minlength=dims[mode]))])
            assert np.array_equal(ptr.cpu().numpy(), want)

    def test_hot_copy_plan(self, at):
        """alto_hot_copies: per hot row 2^lg copies with 2^lg * HOT_BOUND >=
        estimated merges (lg <= HOT_MAX_LG), laid out slot by slot."""
        import importlib

        import torch

        mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
        st = synth.make_tensor(2, nnz=400_000)
        alto = at.build_alto(at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64)), dtype="float32")
        for mode in range(3):
            hp = mk.hot_plan_ms(alto, mode, 16, torch.float32)
            assert hp is not None
            code, rows, n, base, buf = hp
            code, rows, base = code.cpu().numpy(), rows.cpu().numpy()[:n], base.cpu().numpy()
            counts = np.bincount(st.coords[:, mode], minlength=st.config.dims[mode])
            T = mk.ms_tile(alto)
            ntiles = -(-alto.nnz // T)
            assert base[0] == 0 and buf.numel() == base[n] * 16 and float(buf.abs().sum()) == 0.0
            for s, r in enumerate(rows):
                c = int(counts[r])
                est = (c // (T // 8) + 2) if mk.MS_ORDER == 1 else min(c, ntiles) + c // (T // 8)
                lg = int(code[r]) & 31
                assert code[r] >> 5 == base[s] and base[s + 1] - base[s] == 1 << lg
                assert lg == mk.HOT_MAX_LG or (1 << lg) * mk.HOT_BOUND >= est
                assert lg == 0 or (1 << (lg - 1)) * mk.HOT_BOUND < est
            others = np.ones(len(code), bool)
            others[rows] = False
            assert (code[others] == -1).all()

    @pytest.mark.parametrize("cfg,rank", [(2, 16), (3, 32), ("wide", 16), (1, 16)])
    def test_deterministic_fixed_point(self, at, monkeypatch, cfg, rank):
        """Fixed-point streaming mode (used for Buffered / seq when rows are
        long): bitwise identical across runs, ~1e-13 from the fp64 oracle."""
        import importlib

        mk = importlib.import_module("paper_2102_10245_b200.mttkrp")

        monkeypatch.setattr(mk, "EXACT_MAX_RUN", 0)  # force the fixed-point path at test size
        st = synth.make_tensor(self.WIDE if cfg == "wide" else cfg, nnz=150_000)
        dims = st.config.dims
        fp32 = st.config.value_dtype == "float32"
        alto = at.build_alto(at.CooTensor(dims, st.coords, st.values.astype(np.float64)),
                             dtype="float32" if fp32 else "float64")
        factors = seeded_factors(dims, rank, 21)
        for mode in range(len(dims)):
            a = at.mttkrp_seq(alto, factors, mode)
            b = at.mttkrp_seq(alto, factors, mode)
            assert np.array_equal(a, b)
            ref = orc.mttkrp_coo(st.coords, st.values.astype(np.float64), factors, mode)
            assert rel_error(a, ref) <= 1e-12, rel_error(a, ref)
            parts = at.partition(alto, 6)
            plan = at.plan_conflicts(alto, parts, mode, force_strategy=at.Strategy.BUFFERED)
            c = at.mttkrp_par(alto, parts, plan, factors, mode, workers=3)
            assert np.array_equal(a, c)

    def test_accumulates_into_out(self, at):
        from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_stream

        t = at.random_tensor((40, 30, 20), 3000, seed=5)
        alto = at.build_alto(t)
        fdev = factors_to_device(seeded_factors(t.dims, 16, 1))
        a = mttkrp_stream(alto, fdev, 0)
        b = mttkrp_stream(alto, fdev, 0, out=a.clone(), zero_out=False)
        assert rel_error(b.cpu().numpy(), 2 * a.cpu().numpy()) <= 1e-15

    def test_large_linearity(self, at):
        """Size-independent property at 5M elements on the cfg2 law:
        MTTKRP(2X) == 2 MTTKRP(X) and mode sums are consistent."""
        import torch

        from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_stream

        st = synth.make_tensor(2, nnz=5_000_000)
        coo = at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64))
        alto = at.build_alto(coo, dtype="float32")
        ones = [torch.ones((d, 16), dtype=torch.float32, device="cuda") for d in st.config.dims]
        total = float(alto.vals.double().sum())
        for mode in range(3):
            out = mttkrp_stream(alto, ones, mode)
            # all-ones factors: every column sums to sum(values) (test_mttkrp.py:45-52 idea)
            col = out.sum(0).cpu().numpy()
            assert np.allclose(col, total, rtol=1e-6)
        f = factors_to_device(seeded_factors(st.config.dims, 16, 3), torch.float32)
        two = at.AltoTensor(alto.layout, alto.keys, alto.vals * 2)
        a = mttkrp_stream(alto, f, 1)
        b = mttkrp_stream(two, f, 1)
        assert rel_error(b.cpu().numpy(), 2 * a.cpu().numpy()) <= 1e-6


def test_pinned_inputs_async_upload(at):
    """Pinned host torch factors are uploaded on a side stream that overlaps
    the previous call's kernels; back-to-back calls (no host sync between)
    give the results of NumPy inputs (to float32-atomic rounding: the Atomic
    plan's merge order is not fixed)."""
    import torch

    st = synth.make_tensor(2, nnz=200_000)
    dims = st.config.dims
    alto = at.build_alto(at.CooTensor(dims, st.coords, st.values.astype(np.float64)), dtype="float32")
    parts = at.partition(alto, 8)
    rng = np.random.default_rng(9)
    sets = [[rng.random((d, 16)).astype(np.float32) for d in dims] for _ in range(4)]
    plans = [at.plan_conflicts(alto, parts, n, force_strategy=at.Strategy.ATOMIC) for n in range(3)]
    flagged = [at.apply_boundary_flags(alto, p) if p.flag_bit is not None else alto for p in plans]
    outs = []
    for fs in sets:
        pinned = [torch.from_numpy(f).pin_memory() for f in fs]
        for n in range(3):
            outs.append(at.mttkrp_par(flagged[n], parts, plans[n], pinned, n))
    torch.cuda.synchronize()
    k = 0
    for fs in sets:
        for n in range(3):
            ref = at.mttkrp_par(flagged[n], parts, plans[n], fs, n)
            assert rel_error(outs[k].cpu().numpy(), ref) <= 1e-6
            k += 1


def test_fp32_accuracy_at_scale(at):
    """Size-independent property at 20M elements of the cfg5 law (Zipf 1.05,
    128-bit keys): the float32 streaming result (hot rows merged into
    per-row replicated copies with bounded merges) stays within 1e-6 of the
    int64 fixed-point result, which is ~1e-13 from the exact sums."""
    import importlib

    import torch

    from paper_2102_10245_b200.format import build_alto_device
    from paper_2102_10245_b200.layout import build_masks

    mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
    c = synth.CONFIGS[5]
    coords, vals = synth.make_tensor_device(5, nnz=20_000_000)
    alto = build_alto_device(build_masks(c.dims), coords, vals)
    del coords
    rng = np.random.default_rng(3)
    f = mk.factors_to_device([rng.random((d, 16)).astype(np.float32) for d in c.dims])
    for mode in range(3):
        exact = mk.mttkrp_det(alto, f, mode)
        fast = mk.mttkrp_stream(alto, f, mode, out_dtype=torch.float32).double()
        assert float((fast - exact).norm() / exact.norm()) <= 1e-6
        del exact, fast
        torch.cuda.synchronize()


def _installed_reference():
    """The unmodified reference from baseline/_ref (bench.py's reference arm),
    or None; this test is skipped where it was not installed."""
    import importlib
    import os
    import sys

    ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "altotensor")):
        return None
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    return importlib.import_module("altotensor")


@pytest.mark.parametrize("cfg,nnz", [(1, 100_000), (2, 300_000), (4, 200_000)])
def test_live_reference_bitwise(at, cfg, nnz):
    """Device Buffered mttkrp_par == the installed reference's mttkrp_par,
    bit for bit, on a same-law sample of a BASELINE config (reference
    mttkrp.py:132-175, fixed partition count => deterministic)."""
    ref = _installed_reference()
    if ref is None:
        pytest.skip("baseline/_ref not installed")
    st = synth.make_tensor(cfg, nnz=nnz)
    dims, rank = st.config.dims, st.config.rank
    coords, values = st.coords, st.values.astype(np.float64)
    factors = seeded_factors(dims, rank, seed=cfg)
    r_alto = ref.build_alto(ref.CooTensor(dims, coords, values))
    d_alto = at.build_alto(at.CooTensor(dims, coords, values))
    assert np.array_equal(d_alto.indices, r_alto.indices)
    assert np.array_equal(d_alto.values, r_alto.values)
    for mode in range(len(dims)):
        r_parts = ref.partition(r_alto, 16)
        r_plan = ref.plan_conflicts(r_alto, r_parts, mode, force_strategy=ref.Strategy.BUFFERED)
        want = ref.mttkrp_par(r_alto, r_parts, r_plan, factors, mode, 4)
        d_parts = at.partition(d_alto, 16)
        d_plan = at.plan_conflicts(d_alto, d_parts, mode, force_strategy=at.Strategy.BUFFERED)
        got = at.mttkrp_par(d_alto, d_parts, d_plan, factors, mode, workers=4)
        assert np.array_equal(got, want), (cfg, mode, rel_error(got, want))


@pytest.mark.parametrize("cfg,nnz", [(2, 300_000), (4, 200_000), (3, 100_000)])
def test_device_oracle_bitwise_vs_c_oracle(at, cfg, nnz):
    """The drop-in mttkrp_oracle accumulates in input order (np.add.at,
    mttkrp.py:75): bit for bit the C oracle, which is pinned to the reference."""
    from oracle import oracle_c

    st = synth.make_tensor(cfg, nnz=nnz)
    dims, rank = st.config.dims, st.config.rank
    coo = at.CooTensor(dims, st.coords, st.values.astype(np.float64))
    factors = seeded_factors(dims, rank, seed=cfg)
    for mode in range(len(dims)):
        got = at.mttkrp_oracle(coo, factors, mode)
        want = oracle_c.mttkrp_coo(st.coords, st.values.astype(np.float64), factors, mode)
        assert np.array_equal(got, want), (cfg, mode)
