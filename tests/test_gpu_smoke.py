"""The driver's round-end smoke(): runs the in-tree libalto_b200.so on cuda:0
and checks it against the oracle (ALTO build, partition, MTTKRP, CP-ALS,
ingestion, container)."""

import os

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_smoke_runs_on_the_in_tree_library():
    import __graft_entry__

    __graft_entry__.smoke()
    maps = open("/proc/self/maps").read()
    lib = os.path.join(ROOT, "paper_2102_10245_b200", "lib", "libalto_b200.so")
    assert os.path.realpath(lib) in maps, "smoke() did not load the in-tree libalto_b200.so"
