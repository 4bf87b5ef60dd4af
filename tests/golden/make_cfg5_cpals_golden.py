"""Golden CP-ALS fit history on the cfg5 law, produced by the REFERENCE.

Run in the build container (where /root/reference exists):
    python tests/golden/make_cfg5_cpals_golden.py [nnz]
It draws `nnz` (default 20M) distinct nonzeros of BASELINE.json's cfg5 law
(40M x 20M x 1M, Zipf(1.05) on every mode, uniform(0,1) values rounded to
float32) with the repo's seeded NumPy generator (synth.make_tensor(5, nnz)),
runs the unmodified reference's cpd_als (pkg/src/altotensor/cpd.py:184-228)
for 10 iterations at rank 16 with tol=0 (backend "auto", 8 workers, as the
CLI protocol cli.py:198-216 does), and stores fit_history, the final weights
and per-factor column norms in tests/golden/cfg5_cpals_<nnz>.npz, together
with SHA-256 digests of the generated coordinates and values so that the GPU
test can check the box regenerated the identical tensor.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import altotensor as ref  # noqa: E402  (the reference)

from paper_2102_10245_b200 import synth  # noqa: E402  (seeded generator only)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
    t0 = time.time()
    st = synth.make_tensor(5, nnz=nnz)
    t_gen = time.time() - t0
    coo = ref.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64))
    t0 = time.time()
    alto = ref.build_alto(coo)
    t_build = time.time() - t0
    t0 = time.time()
    model = ref.cpd_als(alto, 16, max_iters=10, tol=0.0, seed=0, backend="auto", workers=8)
    t_als = time.time() - t0
    meta = {"cfg": 5, "nnz": nnz, "dims": list(st.config.dims), "rank": 16, "iters": 10, "seed": 0,
            "backend": "auto", "workers": 8, "tensor_seed": st.seed,
            "coords_sha": sha(st.coords), "values_sha": sha(st.values),
            "reference": "altotensor " + ref.__version__, "gen_s": t_gen, "build_s": t_build, "cpd_s": t_als}
    np.savez_compressed(os.path.join(HERE, f"cfg5_cpals_{nnz}.npz"),
                        fit_history=np.asarray(model.fit_history, dtype=np.float64),
                        weights=np.asarray(model.weights, dtype=np.float64),
                        factor_col_norms=np.stack([np.linalg.norm(f, axis=0) for f in model.factors]),
                        meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8))
    print(json.dumps(meta), model.fit_history)


if __name__ == "__main__":
    main()
