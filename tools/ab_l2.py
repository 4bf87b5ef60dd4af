"""A/B: L2 residency policies for the gathered factors of the mode-stream kernel
(MS_L2_HOT_MB: leading bytes of each input factor evict_last, the rest and the
output merges evict_first) vs the default policy.  python tools/ab_l2.py cfg [MB ...]"""
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
    budgets = [float(x) for x in sys.argv[2:]] or [0, 32, 64, 96]
    c = synth.CONFIGS[cfg]
    R = c.rank
    coords, vals = synth.make_tensor_device(cfg)
    lay = build_masks(c.dims)
    alto = build_alto_device(lay, coords, vals)
    del coords
    rng = np.random.default_rng(7)
    f32 = mk.factors_to_device([rng.random((d, R)).astype(np.float32) for d in c.dims])
    ba = alto.nnz * (8 * lay.n_words + 4) + sum(d * R * 4 for d in c.dims)
    ref = None
    for mb in budgets + [budgets[0]]:
        mk.MS_L2_HOT_MB = mb
        res = {"cfg": cfg, "l2_hot_mb": mb, "ms": [], "hot_bytes": []}
        outs = []
        for mode in range(len(c.dims)):
            out = torch.empty((c.dims[mode], R), dtype=torch.float32, device="cuda")
            res["ms"].append(timed(lambda: mk.mttkrp_stream(alto, f32, mode, out=out)))
            res["hot_bytes"].append(mk.l2_hot_bytes(c.dims, mode, R, 4))
            outs.append(mk.mttkrp_stream(alto, f32, mode, out_dtype=torch.float32).double())
        res["frac"] = len(c.dims) * ba / (sum(res["ms"]) * 1e-3) / 1e9 / 6447.5
        if ref is None:
            ref = outs
        res["rel_diff"] = [float((a - b).norm() / b.norm()) for a, b in zip(outs, ref)]
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
