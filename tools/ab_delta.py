"""A/B: mode-stream kernel with one-word delta keys (ALTO_MS_DELTA) vs the
two-word stream on 128-bit layouts, per mode.  python tools/ab_delta.py cfg"""
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


def main():
    cfg = int(sys.argv[1])
    ranks = [int(x) for x in sys.argv[2:]] or [synth.CONFIGS[cfg].rank]
    c = synth.CONFIGS[cfg]
    coords, vals = synth.make_tensor_device(cfg)
    lay = build_masks(c.dims)
    alto = build_alto_device(lay, coords, vals)
    del coords
    for R in ranks:
        if R not in mk.MS_RANKS:
            mk.MS_RANKS = mk.MS_RANKS + (R,)
        rng = np.random.default_rng(7)
        f32 = mk.factors_to_device([rng.random((d, R)).astype(np.float32) for d in c.dims])
        ba = alto.nnz * (8 * lay.n_words + 4) + sum(d * R * 4 for d in c.dims)
        outs = {}
        for delta in (0, 1):
            mk.MS_DELTA = delta
            for k in [k for k in alto._cache if k[0] in ("mstream", "hotms")]:
                del alto._cache[k]
            torch.cuda.empty_cache()
            res = {"cfg": cfg, "rank": R, "delta": delta, "ms": []}
            outs[delta] = []
            for mode in range(len(c.dims)):
                out = torch.empty((c.dims[mode], R), dtype=torch.float32, device="cuda")
                res["ms"].append(timed(lambda: mk.mttkrp_stream(alto, f32, mode, out=out)))
                outs[delta].append(mk.mttkrp_stream(alto, f32, mode, out_dtype=torch.float32).double())
                ms = mk.mode_stream(alto, mode)
                res.setdefault("is_delta", []).append(ms is not None and ms[4] is not None)
            res["frac"] = len(c.dims) * ba / (sum(res["ms"]) * 1e-3) / 1e9 / 6553.0
            print(json.dumps(res), flush=True)
        print(json.dumps({"rel_diff": [float((a - b).norm() / b.norm()) for a, b in zip(outs[1], outs[0])]}))


if __name__ == "__main__":
    main()
