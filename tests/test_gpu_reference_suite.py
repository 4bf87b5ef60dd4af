"""The reference's own test suite (pkg/tests, 177 tests), run UNCHANGED with
layout/format/mttkrp/cpd swapped for the B200 drop-in (SURVEY.md §7.2 item
8; shim: tests/refsuite/shim.py).

The tests are brought along by build() into baseline/_ref/reference_tests
(git-ignored, travels to the GPU box).  Expected exceptions, each justified
in DESIGN.md §2:
  * test_criterion_8_parallel_speedup — a CPU thread-scaling timing check
    of the reference's workers (pkg/tests/test_acceptance.py:227-264);
    `workers` has no effect on the device path.
Everything else must pass.
"""

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
EXPECTED_FAIL = {"test_criterion_8_parallel_speedup"}

pytestmark = pytest.mark.gpu


def test_reference_suite_through_drop_in(tmp_path):
    tests_dir = os.path.join(REF, "reference_tests")
    if not (os.path.isdir(os.path.join(REF, "altotensor")) and os.path.isdir(tests_dir)):
        pytest.skip("baseline/_ref (reference install + its tests) not present")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from refsuite.shim import build_shim

    shim = build_shim(str(tmp_path / "shim"), os.path.join(REF, "altotensor"))
    work = tmp_path / "tests"
    import shutil

    shutil.copytree(tests_dir, work)
    xml = tmp_path / "junit.xml"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([shim, ROOT]))
    r = subprocess.run([sys.executable, "-m", "pytest", str(work), "-q", "-p", "no:cacheprovider",
                        f"--junitxml={xml}", "-o", "addopts=", "--rootdir", str(work)],
                       env=env, capture_output=True, text=True, cwd=str(work), timeout=1800)
    tree = ET.parse(xml)
    failed, passed, skipped = [], 0, 0
    for case in tree.iter("testcase"):
        bad = case.find("failure") is not None or case.find("error") is not None
        if bad:
            failed.append(case.get("name"))
        elif case.find("skipped") is not None:
            skipped += 1
        else:
            passed += 1
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "reference_suite.log"), "w") as f:
        f.write(r.stdout[-20000:] + "\n" + r.stderr[-5000:])
    unexpected = sorted(n for n in failed if n.split("[")[0] not in EXPECTED_FAIL)
    assert passed >= 170, (passed, skipped, failed, r.stdout[-3000:])
    assert not unexpected, (unexpected, r.stdout[-6000:])
