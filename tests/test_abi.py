"""The C-ABI library loads and exports every symbol include/alto_b200.h
declares; host-only queries work without a GPU.  CPU only."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2102_10245_b200 import _lib

HEADER = os.path.join(ROOT, "include", "alto_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(alto_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libalto_b200.so missing: run `make` (or __graft_entry__.build())")
    return _lib.load()


def test_header_parsed():
    names = declared_functions()
    assert "alto_mttkrp" in names and "alto_sort_pairs" in names and len(names) >= 25


def test_every_declared_symbol_exported(lib):
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_functions():
        assert hasattr(raw, name), f"{name} declared in alto_b200.h but not exported"


def test_bindings_cover_header():
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(declared_functions()) <= bound


def test_host_queries(lib):
    assert lib.alto_version() == 1
    assert lib.alto_sort_workspace_bytes(1 << 20, 1, 4) > (1 << 20) * 12
    assert lib.alto_cpd_workspace_bytes(16) >= 256 * 16 * 16 * 8
    assert lib.alto_mttkrp_ntiles(10_000, 1024) == 10
    assert lib.alto_row_index_workspace_bytes(1000, 10) > 8000


def test_tables_bytes_matches_layout(lib):
    from paper_2102_10245_b200.layout import build_masks, c_layout

    lay = build_masks((200_000, 150_000, 100_000))   # cfg2: 53 bits, 7 key bytes
    enc = sum((b + 7) // 8 for b in lay.bits)
    assert lib.alto_tables_bytes(c_layout(lay)) == (enc + 7) * 256 * 8
    wide = build_masks((40_000_000, 20_000_000, 1_000_000))  # cfg5: 71 bits, 128-bit keys
    enc = sum((b + 7) // 8 for b in wide.bits)
    assert lib.alto_tables_bytes(c_layout(wide)) == (enc + 9) * 256 * 16


def test_invalid_argument_maps_to_value_error(lib):
    st = lib.alto_sort_pairs(None, None, 10, 3, 4, 8, None, 0, None)  # n_words=3 is rejected before any CUDA call
    assert st == _lib.ALTO_EINVAL
    with pytest.raises(ValueError):
        _lib.check(st)
