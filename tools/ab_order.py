"""A/B: row-major vs tile-ordered mode streams per mode (mode-stream kernel),
CUDA events, L2 flushed.  python tools/ab_order.py cfg"""
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
    c = synth.CONFIGS[cfg]
    coords, vals = synth.make_tensor_device(cfg)
    lay = build_masks(c.dims)
    alto = build_alto_device(lay, coords, vals)
    del coords
    R = c.rank
    if R not in mk.MS_RANKS:
        mk.MS_RANKS = mk.MS_RANKS + (R,)
    rng = np.random.default_rng(7)
    f32 = mk.factors_to_device([rng.random((d, R)).astype(np.float32) for d in c.dims])
    ref = {}
    for order in (1, 0):
        mk.MS_ORDER = order
        res = {"cfg": cfg, "order": order, "ms": [], "rel_vs_rowmajor": []}
        for mode in range(len(c.dims)):
            for k in [k for k in alto._cache if k[0] in ("mstream", "hotms")]:
                del alto._cache[k]
            torch.cuda.empty_cache()
            out = torch.empty((c.dims[mode], R), dtype=torch.float32, device="cuda")
            res["ms"].append(timed(lambda: mk.mttkrp_stream(alto, f32, mode, out=out)))
            o = mk.mttkrp_stream(alto, f32, mode, out_dtype=torch.float32).double()
            if order == 1:
                ref[mode] = o
            else:
                res["rel_vs_rowmajor"].append(float((o - ref[mode]).norm() / ref[mode].norm()))
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
