"""A/B: mode-stream tile length (MS_TILE) per mode.  python tools/ab_mstile.py cfg"""
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
    alto = build_alto_device(build_masks(c.dims), coords, vals)
    del coords
    rng = np.random.default_rng(7)
    f32 = mk.factors_to_device([rng.random((d, c.rank)).astype(np.float32) for d in c.dims])
    for t in (1024, 2048, 4096, 1024):
        mk.MS_TILE = t
        for k in [k for k in alto._cache if k[0] in ("mstream", "hotms")]:
            del alto._cache[k]
        torch.cuda.empty_cache()
        res = {"cfg": cfg, "ms_tile": t, "ms": []}
        for mode in range(len(c.dims)):
            out = torch.empty((c.dims[mode], c.rank), dtype=torch.float32, device="cuda")
            res["ms"].append(timed(lambda: mk.mttkrp_stream(alto, f32, mode, out=out)))
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
