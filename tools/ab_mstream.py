"""A/B of the MTTKRP kernels on a BASELINE config (ad-hoc measurement, not product):
  python tools/ab_mstream.py [cfg] [nnz] [tiles...]
Times the planned kernel and the mode-stream kernel at several tile lengths
(per mode, CUDA events, L2 flushed between reps) and checks they agree."""
import sys
import time

import numpy as np
import torch

import importlib
mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
from paper_2102_10245_b200 import synth
from paper_2102_10245_b200.format import build_alto_device
from paper_2102_10245_b200.layout import build_masks
from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_stream


def timed(fn, reps=10, flush=None):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    nnz = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else None
    tiles = [int(x) for x in sys.argv[3:]] or [512, 1024, 2048, 4096]
    c = synth.CONFIGS[cfg]
    t0 = time.time()
    coords, vals = synth.make_tensor_device(cfg, nnz=nnz)
    alto = build_alto_device(build_masks(c.dims), coords, vals)
    del coords
    rng = np.random.default_rng(7)
    fd = torch.float32 if c.value_dtype == "float32" else torch.float64
    f = factors_to_device([rng.random((d, c.rank)) for d in c.dims], dtype=fd)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    print(f"cfg{cfg}: nnz {alto.nnz}, build {time.time() - t0:.1f}s", flush=True)
    for mode in range(len(c.dims)):
        exact = mk.mttkrp_det(alto, f, mode)  # int64 fixed point: ~1e-13 of the exact sums
        mk.MS_TILE = 0
        ref = mttkrp_stream(alto, f, mode, out_dtype=fd)
        tp = timed(lambda: mttkrp_stream(alto, f, mode, out=ref, out_dtype=fd), flush=flush)
        ref = mttkrp_stream(alto, f, mode, out_dtype=fd).double()
        line = [f"mode {mode}: planned {tp:.3f} ms (err {float((ref - exact).norm() / exact.norm()):.1e})"]
        ref = exact
        for T in tiles:
            mk.MS_TILE = T
            t1 = time.time()
            mk.mode_stream(alto, mode)
            torch.cuda.synchronize()
            tb = time.time() - t1
            o = mttkrp_stream(alto, f, mode, out_dtype=fd)
            tm = timed(lambda: mttkrp_stream(alto, f, mode, out=o, out_dtype=fd), flush=flush)
            o = mttkrp_stream(alto, f, mode, out_dtype=fd).double()
            err = float((o - ref).norm() / ref.norm())
            line.append(f"T={T}: {tm:.3f} ms (build {tb:.2f}s, rel {err:.1e})")
            for k in [k for k in alto._cache if isinstance(k, tuple) and k[0] == "mstream"]:
                del alto._cache[k]
        mk.MS_TILE = tiles[0]
        for fl in [int(x) for x in __import__("os").environ.get("AB_FLAGS", "").split(",") if x]:
            mk.STREAM_FLAGS = fl
            o = mttkrp_stream(alto, f, mode, out_dtype=fd)
            tm = timed(lambda: mttkrp_stream(alto, f, mode, out=o, out_dtype=fd), flush=flush)
            o = mttkrp_stream(alto, f, mode, out_dtype=fd).double()
            line.append(f"flags {fl}: {tm:.3f} ms (rel {float((o - ref).norm() / ref.norm()):.1e})")
        mk.STREAM_FLAGS = 0
        for fl, nm in ((-1, "tile-order"), (-2, "contiguous-slices")):
            mk.MS_ORDER = 0 if fl == -1 else 1
            mk.MS_RR = 0 if fl == -2 else 1
            for k in [k for k in alto._cache if isinstance(k, tuple) and k[0] in ("mstream", "hotms")]:
                del alto._cache[k]
            mk.STREAM_FLAGS = max(fl, 0)
            o = mttkrp_stream(alto, f, mode, out_dtype=fd)
            tm = timed(lambda: mttkrp_stream(alto, f, mode, out=o, out_dtype=fd), flush=flush)
            o = mttkrp_stream(alto, f, mode, out_dtype=fd).double()
            line.append(f"{nm}: {tm:.3f} ms (rel {float((o - ref).norm() / ref.norm()):.1e})")
        mk.STREAM_FLAGS = 0
        mk.MS_ORDER = 1
        mk.MS_RR = 1
        for k in [k for k in alto._cache if isinstance(k, tuple) and k[0] in ("mstream", "hotms")]:
            del alto._cache[k]
        print("; ".join(line), flush=True)


if __name__ == "__main__":
    main()
