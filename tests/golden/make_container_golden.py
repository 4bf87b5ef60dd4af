"""Golden `.alto` container blobs written by the REFERENCE serializer.

Run in the build container (where /root/reference exists):
    python tests/golden/make_container_golden.py
It imports the unmodified reference package from /root/reference/pkg/src,
serializes seeded tensors (the paper's worked example, a 3-mode random
tensor, a 128-bit-key tensor with boundary flags set, an empty tensor) and
stores the bytes under tests/golden/container_*.alto.  The blobs are the
byte-exact oracle for paper_2102_10245_b200.container (format:
pkg/src/altotensor/container.py:1-19).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import altotensor as at  # noqa: E402  (the reference)
from altotensor.format import Strategy  # noqa: E402


def main() -> None:
    # the worked example (pkg/tests/conftest.py:8-20)
    coords = np.array([[1, 0, 0], [3, 0, 1], [0, 3, 0], [2, 2, 1], [3, 2, 0], [1, 6, 1]], dtype=np.int64)
    ex = at.build_alto(at.CooTensor((4, 8, 2), coords, np.arange(1.0, 7.0)))
    blobs = {"example": at.serialize(ex)}
    blobs["random"] = at.serialize(at.build_alto(at.random_tensor((60, 50, 40), 3000, seed=8)))
    rng = np.random.default_rng(3)
    dims = (1 << 40, 1 << 40)
    c = np.unique(rng.integers(0, dims, size=(50, 2), dtype=np.int64), axis=0)
    wide = at.build_alto(at.CooTensor(dims, c, rng.random(len(c))))
    parts = at.partition(wide, 4)
    plan = at.plan_conflicts(wide, parts, 0, force_strategy=Strategy.ATOMIC)
    blobs["wide_flagged"] = at.serialize(at.apply_boundary_flags(wide, plan))
    blobs["empty"] = at.serialize(at.AltoTensor(at.build_masks((4, 8, 2)), np.empty((0, 1), np.uint64),
                                                np.empty(0)))
    for name, b in blobs.items():
        with open(os.path.join(HERE, f"container_{name}.alto"), "wb") as f:
            f.write(b)
        print(name, len(b), "bytes")


if __name__ == "__main__":
    main()
