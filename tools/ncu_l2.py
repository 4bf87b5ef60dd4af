"""ncu target: the cfg5 mode-stream kernel per mode with and without the L2 residency policies."""
import importlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10245_b200 import synth  # noqa: E402
from paper_2102_10245_b200.format import build_alto_device  # noqa: E402
from paper_2102_10245_b200.layout import build_masks  # noqa: E402

mk = importlib.import_module("paper_2102_10245_b200.mttkrp")


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    c = synth.CONFIGS[cfg]
    R = c.rank
    coords, vals = synth.make_tensor_device(cfg)
    lay = build_masks(c.dims)
    alto = build_alto_device(lay, coords, vals)
    del coords
    rng = np.random.default_rng(7)
    f32 = mk.factors_to_device([rng.random((d, R)).astype(np.float32) for d in c.dims])
    for mb in (0, 64):
        mk.MS_L2_HOT_MB = mb
        for mode in range(len(c.dims)):
            out = torch.empty((c.dims[mode], R), dtype=torch.float32, device="cuda")
            for _ in range(2):
                mk.mttkrp_stream(alto, f32, mode, out=out)
            torch.cuda.synchronize()


if __name__ == "__main__":
    main()
