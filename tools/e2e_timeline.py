"""Timeline of one end-to-end MTTKRP step (bench.py's e2e leg): per mode the
upload, kernel and read-back intervals from CUDA events, plus raw PCIe rates.
python tools/e2e_timeline.py [cfg]"""
import importlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_10245_b200 as at  # noqa: E402
from paper_2102_10245_b200 import synth  # noqa: E402
from paper_2102_10245_b200.format import build_alto_device  # noqa: E402
from paper_2102_10245_b200.layout import build_masks  # noqa: E402

mk = importlib.import_module("paper_2102_10245_b200.mttkrp")


def pcie():
    n = 1 << 30
    x = torch.empty(n, dtype=torch.uint8).pin_memory()
    x2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    y = torch.empty(n, dtype=torch.uint8, device="cuda")
    y2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s2 = torch.cuda.Stream()
    res = {}

    def run(name, fa, fb=None):
        for _ in range(2):
            fa()
            if fb:
                with torch.cuda.stream(s2):
                    fb()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            fa()
            if fb:
                with torch.cuda.stream(s2):
                    fb()
        torch.cuda.synchronize()
        b.record()
        torch.cuda.synchronize()
        res[name] = 4 * n / (a.elapsed_time(b) * 1e-3) / 1e9

    run("h2d_GBs", lambda: y.copy_(x, non_blocking=True))
    run("d2h_GBs", lambda: x2.copy_(y2, non_blocking=True))
    run("bidir_each_GBs", lambda: y.copy_(x, non_blocking=True), lambda: x2.copy_(y2, non_blocking=True))
    return res


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    print(json.dumps({"pcie": pcie()}), flush=True)
    c = synth.CONFIGS[cfg]
    R = c.rank
    coords, vals = synth.make_tensor_device(cfg)
    lay = build_masks(c.dims)
    alto = build_alto_device(lay, coords, vals)
    del coords
    rng = np.random.default_rng(7)
    fpin = [torch.from_numpy(rng.random((d, R)).astype(np.float32)).pin_memory() for d in c.dims]
    opin = [torch.empty((d, R), dtype=torch.float64).pin_memory() for d in c.dims]
    mk.OVERLAP_UPLOADS = True
    parts = at.partition(alto, 16)
    plans = [at.plan_conflicts(alto, parts, n) for n in range(len(c.dims))]
    d2h = torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def step(ev=None):
        for n in range(len(c.dims)):
            o = at.mttkrp_par(alto, parts, plans[n], fpin, n, workers=1)
            if ev is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(cur)
                ev.append(("kernel_done", n, e))
            d2h.wait_stream(cur)
            with torch.cuda.stream(d2h):
                opin[n].copy_(o, non_blocking=True)
                if ev is not None:
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(d2h)
                    ev.append(("d2h_done", n, e))
            o.record_stream(d2h)
        torch.cuda.synchronize()

    for _ in range(2):
        step()
    ev = []
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(cur)
    step(ev)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record(cur)
    torch.cuda.synchronize()
    print(json.dumps({"cfg": cfg, "step_ms": t0.elapsed_time(t1),
                      "events_ms": [(k, n, round(t0.elapsed_time(e), 2)) for k, n, e in ev]}), flush=True)
    # steady state over 3 steps
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    for _ in range(3):
        step()
    b.record(cur)
    torch.cuda.synchronize()
    print(json.dumps({"steady_ms_per_step": a.elapsed_time(b) / 3}))


if __name__ == "__main__":
    main()
