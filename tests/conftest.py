"""Shared fixtures.  `gpu` marks tests that need a B200 (run with -m gpu)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

# The worked example of the paper (pkg/tests/conftest.py:8-20).
EXAMPLE_DIMS = (4, 8, 2)
EXAMPLE_COORDS = np.array([[1, 0, 0], [3, 0, 1], [0, 3, 0], [2, 2, 1], [3, 2, 0], [1, 6, 1]])
EXAMPLE_VALUES = np.arange(1.0, 7.0)
EXAMPLE_LINEAR = [2, 11, 20, 25, 26, 51]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built libalto_b200.so")


def load_golden(name: str):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    data = {k: z[k] for k in z.files}
    meta = json.loads(bytes(data.pop("meta")).decode())
    return data, meta


GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN)
                      if f.endswith(".npz") and not f.startswith(("coo_", "cfg5_cpals")))


def rel_error(out, ref) -> float:
    denom = float(np.linalg.norm(ref))
    diff = float(np.linalg.norm(np.asarray(out) - np.asarray(ref)))
    return diff / denom if denom else diff


@pytest.fixture
def at():
    import paper_2102_10245_b200 as pkg

    return pkg


@pytest.fixture
def example_coo(at):
    return at.CooTensor(EXAMPLE_DIMS, EXAMPLE_COORDS, EXAMPLE_VALUES)


@pytest.fixture
def example_alto(at, example_coo):
    return at.build_alto(example_coo)
