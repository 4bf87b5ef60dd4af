"""Randomised cross-check of every MTTKRP engine against the NumPy oracle
(tools/stress_mttkrp.py): random orders 3-5, ranks including 5/8/12/64 (generic
kernel), both value dtypes, 64- and 128-bit layouts, sizes around tile and
warp-step boundaries, rows hot enough for the replicated-copy plans."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("seed", [3, 11])
def test_random_shapes_all_engines(seed):
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_mttkrp.py"), "14", str(seed)],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0 and "stress ok" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])


def test_random_shapes_cpals_all_backends():
    """tools/stress_cpals.py: random small tensors (orders 3-5, ranks 3/4/7/16/32, both dtypes), every
    CP-ALS backend vs the oracle's fit history (1e-9 relative in float64, 2e-5 in float32)."""
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_cpals.py"), "16", "7"],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0 and "cpals stress ok" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])

