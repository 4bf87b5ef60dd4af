"""A/B: blocked mode-stream kernel (MS_RR = 3: broadcast vector loads, no
shuffles, forced for every shape) vs the round-robin cooperative-decode kernel
(MS_RR = 1), per mode.
python tools/ab_blk.py cfg [rank ...]"""
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
        rng = np.random.default_rng(7)
        f32 = mk.factors_to_device([rng.random((d, R)).astype(np.float32) for d in c.dims])
        ba = alto.nnz * (8 * lay.n_words + 4) + sum(d * R * 4 for d in c.dims)
        outs = {}
        for rr, fl in ((1, 0), (3, 0), (1, 0), (3, 0)):
            mk.MS_RR = rr
            mk.STREAM_FLAGS = fl
            for k in [k for k in alto._cache if k[0] in ("mstream", "hotms")]:
                del alto._cache[k]
            torch.cuda.empty_cache()
            res = {"cfg": cfg, "rank": R, "ms_rr": rr, "flags": fl, "ms": []}
            outs[rr] = []
            for mode in range(len(c.dims)):
                out = torch.empty((c.dims[mode], R), dtype=torch.float32, device="cuda")
                res["ms"].append(timed(lambda: mk.mttkrp_stream(alto, f32, mode, out=out)))
                outs[rr].append(mk.mttkrp_stream(alto, f32, mode, out_dtype=torch.float32).double())
            res["frac"] = len(c.dims) * ba / (sum(res["ms"]) * 1e-3) / 1e9 / 6447.5
            print(json.dumps(res), flush=True)
        print(json.dumps({"rel_diff": [float((a - b).norm() / b.norm()) for a, b in zip(outs[3], outs[1])]}))


if __name__ == "__main__":
    main()
