"""Randomised CP-ALS cross-check: random small tensors (orders 3-5, ranks incl. 3/4/7/16/32,
both value dtypes), every backend, fit history and weights against the NumPy oracle's cpd_als.
python tools/stress_cpals.py [cases] [seed]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2102_10245_b200 as at  # noqa: E402
from oracle import alto_oracle as orc  # noqa: E402  (checker only)
from paper_2102_10245_b200 import synth  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    worst = {}
    for c in range(cases):
        order = int(rng.integers(3, 6))
        dims = tuple(int(rng.integers(3, 200)) for _ in range(order))
        space = float(np.prod([float(d) for d in dims]))
        nnz = int(rng.choice([50, 500, 3000, 20000]))
        laws = tuple((("zipf", 1.1) if rng.random() < 0.5 else ("uniform", 0)) for _ in range(order))
        f32 = rng.random() < 0.5
        rank = int(rng.choice([3, 4, 7, 16, 32]))
        # keep the normal equations well conditioned (a tensor with fewer nonzeros than rank x modes makes
        # the Hadamard of Grams singular: the ridge-retry result then depends on the Cholesky's rounding)
        nnz = max(nnz, 100 * rank)
        nnz = int(min(nnz, max(4, space // 3)))
        cfg = synth.SynthConfig(f"cfg{c + 300}", dims, 0, laws, "uniform01", "float32" if f32 else "float64", rank)
        st = synth.make_tensor(cfg, nnz=nnz, seed=int(rng.integers(1 << 30)))
        vals = st.values.astype(np.float32).astype(np.float64) if f32 else st.values.astype(np.float64)
        alto = at.build_alto(at.CooTensor(dims, st.coords, vals), dtype="float32" if f32 else "float64")
        lay = orc.build_layout(dims)
        words, ov = orc.build(lay, st.coords, vals)
        seed = int(rng.integers(1000))
        _f, w_ref, hist, _ = orc.cpd_als(lay, words, ov, rank, max_iters=3, tol=0.0, seed=seed)
        for be in at.BACKENDS:
            m = at.cpd_als(alto, rank=rank, max_iters=3, tol=0.0, seed=seed, backend=be, workers=2, partitions=4)
            h = np.asarray(m.fit_history)
            err = float(np.max(np.abs(h - hist) / np.maximum(np.abs(hist), 1e-3)))
            tol = 2e-5 if f32 else 1e-9
            worst[(be, f32)] = max(worst.get((be, f32), 0.0), err)
            if not err <= tol or len(h) != len(hist):
                print("FAIL", c, dims, nnz, laws, "f32" if f32 else "f64", rank, be, err, h, hist, flush=True)
                sys.exit(1)
    print("cpals stress ok:", cases, "cases; worst fit error", {f"{k[0]}/{'f32' if k[1] else 'f64'}": float("%.2e" % v)
                                                                for k, v in worst.items()})


if __name__ == "__main__":
    main()
