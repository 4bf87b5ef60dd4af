"""Randomised cross-check of every MTTKRP engine against the NumPy oracle on small
tensors of random shape (orders 3-5, ranks incl. non-powers of two, both value
dtypes, skewed and uniform laws, sizes around tile boundaries).
python tools/stress_mttkrp.py [cases] [seed]"""
import importlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2102_10245_b200 as at  # noqa: E402
from oracle import alto_oracle as orc  # noqa: E402  (checker only)
from paper_2102_10245_b200 import synth  # noqa: E402

mk = importlib.import_module("paper_2102_10245_b200.mttkrp")


def rel(a, b):
    n = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / n) if n else float(np.linalg.norm(a - b))


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    worst = {}
    for c in range(cases):
        order = int(rng.integers(3, 6))
        big = rng.random() < 0.3  # some 128-bit layouts
        dims = tuple(int(rng.integers(2, 1 << (int(rng.integers(18, 24)) if big else int(rng.integers(2, 12)))))
                     for _ in range(order))
        space = float(np.prod([float(d) for d in dims]))
        nnz = int(min(rng.choice([1, 7, 31, 32, 33, 127, 128, 129, 1000, 4097, 20000, 70001]), max(1, space // 2)))
        laws = tuple((("zipf", 1.1) if rng.random() < 0.5 else ("uniform", 0)) for _ in range(order))
        f32 = rng.random() < 0.6
        rank = int(rng.choice([16, 32, 16, 32, 8, 64, 5, 12]))
        cfg = synth.SynthConfig(f"cfg{c + 100}", dims, 0, laws, "uniform_pm1", "float32" if f32 else "float64", rank)
        st = synth.make_tensor(cfg, nnz=nnz, seed=int(rng.integers(1 << 30)))
        vals = st.values.astype(np.float32).astype(np.float64) if f32 else st.values.astype(np.float64)
        alto = at.build_alto(at.CooTensor(dims, st.coords, vals), dtype="float32" if f32 else "float64")
        fdt = np.float32 if f32 else np.float64
        fac = [rng.random((d, rank)).astype(fdt) for d in dims]
        fdev = mk.factors_to_device(fac)
        f64 = [f.astype(np.float64) for f in fac]
        tol = 2e-5 if f32 else 1e-11
        for mode in range(order):
            ref = orc.mttkrp_coo(st.coords, vals, f64, mode)
            got = {"stream": mk.mttkrp_stream(alto, fdev, mode),
                   "fast": mk.mttkrp_stream(alto, fdev, mode, planned=False),
                   "api": torch.as_tensor(at.mttkrp(alto, [torch.from_numpy(f).cuda() for f in f64], mode, partitions=4))}
            if rank in (16, 32) and max(alto.layout.bits) <= 31:
                got["alto"] = mk.mttkrp_stream(alto, fdev, mode, planned="pos")
            if f32:
                got["stream32"] = mk.mttkrp_stream(alto, fdev, mode, out_dtype=torch.float32)
            p = mk.mttkrp_pull(alto, fdev, mode)
            if p is not None:
                got["pull"] = p
            for k, v in got.items():
                e = rel(v.double().cpu().numpy(), ref)
                t = 1e-10 if k == "api" and not f32 else (1e-10 if k == "api" else tol)
                worst[k] = max(worst.get(k, 0.0), e)
                if not e <= t:
                    print("FAIL", c, dims, nnz, laws, "f32" if f32 else "f64", rank, "mode", mode, k, e, flush=True)
                    sys.exit(1)
        torch.cuda.synchronize()
    print("stress ok:", cases, "cases; worst relative error per engine", {k: float("%.2e" % v) for k, v in worst.items()})


if __name__ == "__main__":
    main()
