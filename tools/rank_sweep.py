"""Rank-specialisation sweep (paper PAPER.md:475-511): per-mode
MTTKRP time at R = 8/16/32/64 for the rank-specialised kernels (K8/K9 pull
engine, templated on R; the mode-stream kernel at R=16) against the generic
streaming kernel (runtime rank, ALTO_STREAM_GENERIC), float32, CUDA events.
  python tools/rank_sweep.py [cfg]"""
import importlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10245_b200 import synth  # noqa: E402
from paper_2102_10245_b200.format import build_alto_device  # noqa: E402
from paper_2102_10245_b200.layout import build_masks  # noqa: E402

mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ab_pull import timed  # noqa: E402

GENERIC = 128  # ALTO_STREAM_GENERIC


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    c = synth.CONFIGS[cfg]
    coords, vals = synth.make_tensor_device(cfg)
    lay = build_masks(c.dims)
    alto = build_alto_device(lay, coords, vals)
    del coords
    for R in (8, 16, 32, 64):
        rng = np.random.default_rng(R)
        f = mk.factors_to_device([rng.random((d, R)).astype(np.float32) for d in c.dims])
        res = {"cfg": cfg, "rank": R, "ms": {}}
        N = len(c.dims)
        outs = [torch.empty((d, R), dtype=torch.float32, device="cuda") for d in c.dims]
        res["ms"]["pull_specialised"] = sum(timed(lambda: mk.mttkrp_pull(alto, f, n, out=outs[n])) for n in range(N))
        if R == 16:
            res["ms"]["mode_stream_specialised"] = sum(timed(lambda: mk.mttkrp_stream(alto, f, n, out=outs[n]))
                                                       for n in range(N))
        mk.STREAM_FLAGS = GENERIC
        try:
            res["ms"]["generic"] = sum(timed(lambda: mk.mttkrp_stream(alto, f, n, out=outs[n], planned=False))
                                       for n in range(N))
        finally:
            mk.STREAM_FLAGS = 0
        ref = [mk.mttkrp_stream(alto, f, n, planned=False).double() for n in range(N)]
        got = [mk.mttkrp_pull(alto, f, n, out_dtype=torch.float32).double() for n in range(N)]
        res["rel_diff_pull_vs_generic"] = max(float((a - b).norm() / b.norm()) for a, b in zip(got, ref))
        res["nnz_per_s"] = {k: N * alto.nnz / (v * 1e-3) for k, v in res["ms"].items()}
        res["speedup_specialised_vs_generic"] = res["ms"]["generic"] / min(
            v for k, v in res["ms"].items() if k != "generic")
        print(json.dumps(res), flush=True)
        for k in [k for k in alto._cache if k[0] in ("hot", "hotms")]:
            del alto._cache[k]


if __name__ == "__main__":
    main()
