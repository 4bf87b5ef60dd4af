"""Golden COO-ingestion vectors from the REFERENCE (coalesce, parse_tns,
random_tensor).  Run in the build container (where /root/reference exists):
    python tests/golden/make_coo_golden.py
Stores tests/golden/coo_coalesce.npz: seeded duplicate-heavy inputs and the
reference's CooTensor.coalesce() outputs (pkg/src/altotensor/coo.py:97-114),
plus the reference's random_tensor((50, 40, 30), 10000, seed=7)."""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import altotensor as at  # noqa: E402  (the reference)


def main() -> None:
    out = {}
    for k, (dims, m) in enumerate([((4, 4), 40), ((50, 40, 30), 20000), ((7, 3, 5, 2, 4), 5000),
                                   ((1 << 40, 1 << 40, 1 << 30), 3000)]):
        rng = np.random.default_rng(100 + k)
        hi = np.minimum(np.asarray(dims), 6)
        c = rng.integers(0, hi, size=(m, len(dims)), dtype=np.int64)
        if max(dims) > 1 << 20:
            c[::3] = rng.integers(0, dims, size=(len(c[::3]), len(dims)), dtype=np.int64)
        v = rng.standard_normal(m) * 10.0 ** rng.integers(-8, 8, m)
        t = at.CooTensor(dims, c, v).coalesce()
        out[f"dims{k}"] = np.asarray(dims, dtype=np.int64)
        out[f"in_coords{k}"], out[f"in_values{k}"] = c, v
        out[f"coords{k}"], out[f"values{k}"] = t.coords, t.values
    r = at.random_tensor((50, 40, 30), 10000, seed=7)
    out["rand_coords"], out["rand_values"] = r.coords, r.values
    np.savez_compressed(os.path.join(HERE, "coo_coalesce.npz"), **out)
    print({k: v.shape for k, v in out.items() if k.startswith("coords") or k.startswith("rand")})


if __name__ == "__main__":
    main()
