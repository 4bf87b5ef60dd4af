"""CP-ALS parity on BASELINE.json's cfg5 law (the config that specifies
CP-ALS: 10 iterations, rank 16): device cpd_als vs the fp64 fit history the
UNMODIFIED reference produced on a 20M-nonzero sample of the same law
(tests/golden/make_cfg5_cpals_golden.py; reference cpd.py:184-228, backend
"auto", tol=0).  The box regenerates the identical tensor with the seeded
NumPy generator (checked by SHA-256 against the fixture)."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2102_10245_b200 import synth

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg5_cpals_20000000.npz")


@pytest.fixture(scope="module")
def cfg5_sample():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["meta"]).decode())
    st = synth.make_tensor(5, nnz=meta["nnz"])
    assert hashlib.sha256(np.ascontiguousarray(st.coords).tobytes()).hexdigest() == meta["coords_sha"]
    assert hashlib.sha256(np.ascontiguousarray(st.values).tobytes()).hexdigest() == meta["values_sha"]
    return st, meta, {k: z[k] for k in ("fit_history", "weights", "factor_col_norms")}


@pytest.mark.parametrize("dtype,backend,tol", [("float32", "auto", 1e-5), ("float32", "atomic", 1e-5),
                                               ("float64", "auto", 1e-10)])
def test_cfg5_law_cpals_fit_history_vs_reference(at, cfg5_sample, dtype, backend, tol):
    import torch

    st, meta, ref = cfg5_sample
    alto = at.build_alto(at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64)), dtype=dtype)
    model = at.cpd_als(alto, meta["rank"], max_iters=meta["iters"], tol=0.0, seed=meta["seed"], backend=backend,
                       partitions=meta["workers"])
    hist = np.asarray(model.fit_history)
    want = ref["fit_history"]
    assert hist.shape == want.shape
    rel = np.abs(hist - want) / np.abs(want)
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "cfg5_cpals_parity.jsonl"), "a") as f:
        f.write(json.dumps({"nnz": meta["nnz"], "dtype": dtype, "backend": backend, "max_rel_fit": float(rel.max()),
                            "fit": hist.tolist(), "ref_fit": want.tolist(),
                            "weights_rel": float(np.max(np.abs(np.asarray(model.weights) - ref["weights"])
                                                        / np.abs(ref["weights"])))}) + "\n")
    assert rel.max() <= tol, (dtype, backend, rel.max(), hist, want)
    np.testing.assert_allclose(model.weights, ref["weights"], rtol=1e-3 if dtype == "float32" else 1e-8)
    del alto
    torch.cuda.empty_cache()
