"""A/B: raw-key exchange in the cooperative mode-stream kernel (STREAM_FLAGS 256)
vs decoded-record shuffles, per mode.  python tools/ab_rawx.py cfg"""
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
    R = c.rank
    coords, vals = synth.make_tensor_device(cfg)
    lay = build_masks(c.dims)
    alto = build_alto_device(lay, coords, vals)
    del coords
    rng = np.random.default_rng(7)
    f32 = mk.factors_to_device([rng.random((d, R)).astype(np.float32) for d in c.dims])
    ba = alto.nnz * (8 * lay.n_words + 4) + sum(d * R * 4 for d in c.dims)
    outs = {}
    for fl in (0, 256, 0, 256):
        mk.STREAM_FLAGS = fl
        res = {"cfg": cfg, "flags": fl, "ms": []}
        outs[fl] = []
        for mode in range(len(c.dims)):
            out = torch.empty((c.dims[mode], R), dtype=torch.float32, device="cuda")
            res["ms"].append(timed(lambda: mk.mttkrp_stream(alto, f32, mode, out=out)))
            outs[fl].append(mk.mttkrp_stream(alto, f32, mode, out_dtype=torch.float32).double())
        res["frac"] = len(c.dims) * ba / (sum(res["ms"]) * 1e-3) / 1e9 / 6447.5
        print(json.dumps(res), flush=True)
    print(json.dumps({"rel_diff": [float((a - b).norm() / b.norm()) for a, b in zip(outs[256], outs[0])]}))


if __name__ == "__main__":
    main()
