"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden, rel_error
from oracle import alto_oracle as orc
from paper_2102_10245_b200 import synth


def _inputs(data, meta):
    if "coords" in data:
        return data["coords"], data["values"]
    name = meta["name"]
    if name == "cfg1":
        st = synth.make_tensor(1)
    elif name == "cfg2_200k":
        st = synth.make_tensor(2, nnz=200_000)
    else:
        raise KeyError(name)
    return st.coords, st.values.astype(np.float64)


def _factors(data, meta):
    if "factor_0" in data:
        return [data[f"factor_{n}"] for n in range(len(meta["dims"]))]
    rng = np.random.default_rng(meta["fseed"])
    return [rng.random((d, meta["rank"])) for d in meta["dims"]]


def _check_out(data, meta, key, out, exact=True):
    u = np.random.default_rng(99).random(meta["rank"])
    if meta.get("project"):
        ref = data[key + "_proj"]
        got = out @ u
        assert rel_error(got, ref) <= (0 if exact else 1e-12) + 1e-15
        assert abs(np.linalg.norm(out) - float(data[key + "_fro"])) <= 1e-12 * float(data[key + "_fro"])
    elif exact:
        assert np.array_equal(out, data[key]), key
    else:
        assert rel_error(out, data[key]) <= 1e-12, key


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_matches_reference(name):
    data, meta = load_golden(name)
    lay = orc.build_layout(meta["dims"])
    assert list(lay.bits) == meta["bits"]
    assert [list(p) for p in lay.positions] == meta["positions"]
    assert [str(m) for m in lay.masks] == meta["masks"]
    assert (lay.total_bits, lay.width) == (meta["total_bits"], meta["width"])
    coords, values = _inputs(data, meta)
    words, vals = orc.build(lay, coords, values)
    import hashlib

    assert hashlib.sha256(words.tobytes()).hexdigest() == meta["indices_sha"]
    assert hashlib.sha256(vals.tobytes()).hexdigest() == meta["sorted_values_sha"]
    for count in meta["counts"]:
        offs, iv, spans = orc.partition(lay, words, count)
        assert np.array_equal(offs, data[f"L{count}_offsets"])
        assert np.array_equal(iv, data[f"L{count}_intervals"])
        assert [[str(a), str(b)] for a, b in spans] == meta[f"L{count}_spans"]
        for mode in range(len(meta["dims"])):
            for force in ("auto", "atomic", "buffered"):
                key = f"L{count}_m{mode}_{force}"
                want = meta["plans"][key]
                got = orc.plan(lay, words.shape[0], iv, mode, None if force == "auto" else force)
                assert got["strategy"] == want["strategy"]
                assert got["reuse"] == want["reuse"]
                assert got["flag_bit"] == want["flag_bit"]
                ov = None if got["overlaps"] is None else [[list(r) for r in o] for o in got["overlaps"]]
                assert ov == want["overlaps"], key
                if force == "atomic" and got["flag_bit"] is not None:
                    fl = orc.flag(lay, words, offs, mode, got["overlaps"], got["flag_bit"])
                    assert hashlib.sha256(fl.tobytes()).hexdigest() == meta[key + "_flagged_sha"]
    if not meta["with_mttkrp"]:
        return
    factors = _factors(data, meta)
    for mode in range(len(meta["dims"])):
        _check_out(data, meta, f"m{mode}_oracle", orc.mttkrp_coo(coords, values, factors, mode))
        _check_out(data, meta, f"m{mode}_seq", orc.mttkrp_seq(lay, words, vals, factors, mode))
        for count in meta["counts"]:
            offs = data[f"L{count}_offsets"]
            iv = data[f"L{count}_intervals"]
            _check_out(data, meta, f"L{count}_m{mode}_buffered_mttkrp",
                       orc.mttkrp_buffered(lay, words, vals, factors, mode, offs, iv, workers=4))
            p = orc.plan(lay, words.shape[0], iv, mode, "atomic")
            w2 = words if p["flag_bit"] is None else orc.flag(lay, words, offs, mode, p["overlaps"], p["flag_bit"])
            _check_out(data, meta, f"L{count}_m{mode}_atomic_mttkrp",
                       orc.mttkrp_atomic(lay, w2, vals, factors, mode, offs, p["flag_bit"], workers=4), exact=False)
    if "cpd" in meta and "seq" in meta["cpd"]["backends"]:
        c = meta["cpd"]
        _f, w, hist, _ = orc.cpd_als(lay, words, vals, c["rank"], max_iters=c["iters"], tol=0.0, seed=c["seed"])
        np.testing.assert_allclose(hist, data["cpd_seq_fit"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(w, data["cpd_seq_weights"], rtol=1e-12)


def test_worked_example_goldens():
    """The reference's own literal goldens (pkg/tests/test_layout.py:29-34,
    test_format.py:15-16, :57-66, :121-126, :150-156)."""
    lay = orc.build_layout((4, 8, 2))
    assert lay.masks == (0b001010, 0b110100, 0b000001)
    assert orc.build_layout((5, 3, 7)).positions == ((1, 4, 6), (0, 3), (2, 5, 7))
    assert orc.build_layout((4, 4)).positions == ((0, 2), (1, 3))
    assert orc.as_int(orc.encode(orc.build_layout((5, 3, 7)), [[4, 2, 6]])[0]) == 232
    coords = np.array([[1, 0, 0], [3, 0, 1], [0, 3, 0], [2, 2, 1], [3, 2, 0], [1, 6, 1]])
    words, _ = orc.build(lay, coords, np.arange(1.0, 7.0))
    assert [orc.as_int(r) for r in words] == [2, 11, 20, 25, 26, 51]
    offs, iv, spans = orc.partition(lay, words, 2)
    assert offs.tolist() == [0, 3, 6] and spans == ((2, 20), (25, 51))
    assert iv.tolist() == [[[0, 3], [0, 3], [0, 1]], [[1, 3], [2, 6], [0, 1]]]
    p = orc.plan(lay, 6, iv, 0)
    assert p["overlaps"] == (((1, 3),), ((1, 3),)) and p["flag_bit"] == 6
    assert orc.read_flags(orc.flag(lay, words, offs, 0, p["overlaps"], 6), 6).tolist() == [
        True, True, False, True, True, True]
