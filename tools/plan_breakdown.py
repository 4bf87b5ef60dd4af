"""Where the mode-stream plan build goes (per mode): packed keys, row index, hot slots, hot copies, stream.
python tools/plan_breakdown.py [cfg]"""
import importlib
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10245_b200 import synth  # noqa: E402
from paper_2102_10245_b200.format import build_alto_device  # noqa: E402
from paper_2102_10245_b200.layout import build_masks  # noqa: E402

mk = importlib.import_module("paper_2102_10245_b200.mttkrp")


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    c = synth.CONFIGS[cfg]
    coords, vals = synth.make_tensor_device(cfg)
    alto = build_alto_device(build_masks(c.dims), coords, vals)
    del coords
    for rep in range(2):
        alto._cache.clear()
        torch.cuda.empty_cache()
        res = {"cfg": cfg, "rep": rep}
        _, res["packed_keys_ms"] = timed(lambda: mk.packed_keys(alto))
        for mode in range(len(c.dims)):
            _, a = timed(lambda: mk.row_ptr(alto, mode))
            _, b = timed(lambda: mk.hot_slots(alto, mode))
            _, d = timed(lambda: mk.hot_plan_ms(alto, mode, c.rank, torch.float32))
            _, e = timed(lambda: mk.mode_stream(alto, mode, rank=c.rank))
            res[f"mode{mode}"] = {"row_ptr_ms": round(a, 2), "hot_slots_ms": round(b, 2), "hot_copies_ms": round(d, 2),
                                  "mode_stream_ms": round(e, 2)}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
