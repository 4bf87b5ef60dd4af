"""`.alto` container: byte-identical to the reference
serializer (golden blobs from tests/golden/make_container_golden.py, which
ran the unmodified reference), the reference's validation cases
(pkg/tests/test_format.py:214-294), and file streaming to / from HBM."""

import os

import numpy as np
import pytest

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")
MAGIC = b"ALTO"


def blob(name):
    return open(os.path.join(GOLD, f"container_{name}.alto"), "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["example", "random", "wide_flagged", "empty"])
def test_golden_round_trip(at, name, tmp_path):
    """deserialize(reference bytes) -> serialize gives the same bytes; the file
    path (chunked device streaming) too, with tiny chunks to cross boundaries."""
    import importlib

    ct = importlib.import_module("paper_2102_10245_b200.container")
    data = blob(name)
    t = at.deserialize(data)
    assert at.serialize(t) == data
    path = str(tmp_path / "t.alto")
    old = ct.CHUNK_BYTES
    try:
        ct.CHUNK_BYTES = 24  # many chunks, both staging buffers reused
        at.write_alto(t, path)
        assert open(path, "rb").read() == data
        back = at.read_alto(path)
    finally:
        ct.CHUNK_BYTES = old
    assert np.array_equal(back.indices, t.indices) and np.array_equal(back.values, t.values)
    assert back.layout == t.layout


@pytest.mark.gpu
def test_matches_reference_build(at, example_coo):
    """Our build_alto of the worked example serializes to the reference's bytes."""
    assert at.serialize(at.build_alto(example_coo)) == blob("example")


@pytest.mark.gpu
def test_float32_storage(at, tmp_path):
    """float32 device values widen exactly on write; dtype='float32' narrows on read."""
    import torch

    from paper_2102_10245_b200 import synth

    st = synth.make_tensor(2, nnz=50_000)
    coo = at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64))
    t32 = at.build_alto(coo, dtype="float32")
    path = str(tmp_path / "c.alto")
    at.write_alto(t32, path)
    back = at.read_alto(path, dtype="float32")
    assert back.vals.dtype == torch.float32
    assert torch.equal(back.vals, t32.vals) and torch.equal(back.keys, t32.keys)
    assert open(path, "rb").read() == at.serialize(t32)
    with pytest.raises(ValueError):
        at.read_alto(path, dtype="int8")


class TestValidation:
    """Malformed containers are rejected before any device work (CPU-only)."""

    def test_bad_magic(self, at):
        b = bytearray(blob("example"))
        b[0] = ord("X")
        with pytest.raises(at.ContainerError, match="magic"):
            at.deserialize(bytes(b))

    def test_bad_version(self, at):
        b = bytearray(blob("example"))
        b[4] = 9
        with pytest.raises(at.ContainerError, match="version"):
            at.deserialize(bytes(b))

    @pytest.mark.parametrize("w", [32, 128])
    def test_bad_width(self, at, w):
        b = bytearray(blob("example"))
        b[6] = w
        with pytest.raises(at.ContainerError, match="width"):
            at.deserialize(bytes(b))

    def test_truncation(self, at, tmp_path):
        data = blob("example")
        for cut in (2, 6, 20, len(data) - 1):
            with pytest.raises(at.ContainerError, match="truncated|missing"):
                at.deserialize(data[:cut])
            p = str(tmp_path / f"c{cut}.alto")
            open(p, "wb").write(data[:cut])
            with pytest.raises(at.ContainerError, match="truncated|missing"):
                at.read_alto(p)

    def test_trailing_data(self, at, tmp_path):
        with pytest.raises(at.ContainerError, match="trailing"):
            at.deserialize(blob("example") + b"\x00")
        p = str(tmp_path / "t.alto")
        open(p, "wb").write(blob("example") + b"\x00")
        with pytest.raises(at.ContainerError, match="trailing"):
            at.read_alto(p)

    def test_corrupted_mask(self, at):
        b = bytearray(blob("example"))
        b[8 + 3 * 8 + 8] ^= 0xFF
        with pytest.raises(at.ContainerError, match="mask"):
            at.deserialize(bytes(b))

    def test_is_value_error(self, at):
        assert issubclass(at.ContainerError, ValueError)


@pytest.mark.gpu
def test_out_of_range_coordinate_rejected(at, tmp_path):
    """A key whose decoded coordinate is >= the mode extent (the masks admit
    up to 2^b_n - 1) raises ContainerError on read, before any kernel can
    use it as a row (advisor finding: corrupt .alto files)."""
    coo = at.CooTensor((5, 3, 7), np.array([[4, 2, 6], [0, 0, 0]]), np.array([1.0, 2.0]))
    blob = bytearray(at.serialize(at.build_alto(coo)))
    lay = at.build_masks((5, 3, 7))
    bad = at.linearize(lay, (4, 2, 6)) | lay.masks[0]  # mode-0 coordinate 7 >= 5
    nnz, nw = 2, 1
    off = len(blob) - nnz * 8 - nnz * nw * 8
    words = np.frombuffer(bytes(blob[off:off + nnz * 8]), dtype="<u8").copy()
    words[np.argmax(words)] = bad
    blob[off:off + nnz * 8] = words.astype("<u8").tobytes()
    with pytest.raises(at.ContainerError, match="out of range"):
        at.deserialize(bytes(blob))
    p = tmp_path / "bad.alto"
    p.write_bytes(bytes(blob))
    with pytest.raises(at.ContainerError, match="out of range"):
        at.read_alto(str(p))
