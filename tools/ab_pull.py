"""A/B timing: mode-stream kernel (mttkrp_stream) vs the K8/K9 pull engine
(Buffered and Atomic) per mode, CUDA events, L2 flushed between reps.
  python tools/ab_pull.py [cfg ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10245_b200 import synth  # noqa: E402
from paper_2102_10245_b200.format import build_alto_device  # noqa: E402
from paper_2102_10245_b200.layout import build_masks  # noqa: E402
import importlib  # noqa: E402

mk = importlib.import_module("paper_2102_10245_b200.mttkrp")

PEAK = 6553.0


def timed(fn, reps=10):
    l2 = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        l2.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    cfgs = [int(x) for x in sys.argv[1:]] or [2, 4, 5]
    for cfg in cfgs:
        c = synth.CONFIGS[cfg]
        coords, vals = synth.make_tensor_device(cfg)
        lay = build_masks(c.dims)
        alto = build_alto_device(lay, coords, vals)
        del coords
        rng = np.random.default_rng(7)
        f32 = mk.factors_to_device([rng.random((d, c.rank)).astype(np.float32) for d in c.dims])
        f64 = [f.double() for f in f32]
        kb = 8 * lay.n_words
        for mode in range(len(c.dims)):
            ba = alto.nnz * (kb + 4) + sum(d * c.rank * 4 for d in c.dims)
            out32 = torch.empty((c.dims[mode], c.rank), dtype=torch.float32, device="cuda")
            out64 = torch.empty((c.dims[mode], c.rank), dtype=torch.float64, device="cuda")
            res = {"cfg": cfg, "mode": mode}
            res["mstream_f32"] = timed(lambda: mk.mttkrp_stream(alto, f32, mode, out=out32))
            res["pull_buf_f32"] = timed(lambda: mk.mttkrp_pull(alto, f32, mode, out=out32))
            res["pull_atomic_f32"] = timed(lambda: mk.mttkrp_pull(alto, f32, mode, out=out32, atomic=True))
            res["pull_buf_f64fac"] = timed(lambda: mk.mttkrp_pull(alto, f64, mode, out=out64))
            a = mk.mttkrp_stream(alto, f32, mode, out=out32).double()
            b = mk.mttkrp_pull(alto, f32, mode).double()
            res["rel_diff_pull_vs_stream"] = float((a - b).norm() / b.norm())
            res["frac"] = {k: ba / (v * 1e-3) / 1e9 / PEAK for k, v in res.items() if k.endswith(("f32", "fac"))}
            print(json.dumps(res), flush=True)
            alto._cache.clear()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
