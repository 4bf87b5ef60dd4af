"""Ad-hoc measurements used for DESIGN.md (not part of the product):
  python tools/measure_engines.py exact  [nnz]      exact-order engine vs streaming on the cfg2 law
  python tools/measure_engines.py cpals5 [nnz] [it]  CP-ALS on the cfg5 law (128-bit keys)"""
import sys
import time

import numpy as np
import torch

import paper_2102_10245_b200 as at
from paper_2102_10245_b200 import synth
from paper_2102_10245_b200.format import build_alto_device
from paper_2102_10245_b200.layout import build_masks
from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_det, mttkrp_exact, mttkrp_stream


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def exact(nnz, exact_too=True):
    cfg = synth.CONFIGS[2]
    coords, vals = synth.make_tensor_device(2, nnz=nnz)
    alto = build_alto_device(build_masks(cfg.dims), coords, vals)
    rng = np.random.default_rng(7)
    f = factors_to_device([rng.random((d, 16)).astype(np.float32) for d in cfg.dims])
    for mode in range(3):
        te = timed(lambda: mttkrp_exact(alto, f, mode), reps=1) if exact_too else float("nan")
        ts = timed(lambda: mttkrp_stream(alto, f, mode, out_dtype=torch.float32))
        td = timed(lambda: mttkrp_det(alto, f, mode))
        print(f"mode {mode}: exact-order engine {te:.1f} ms, deterministic fixed-point {td:.2f} ms, "
              f"streaming (f32 out) {ts:.2f} ms", flush=True)


def cpals5(nnz, iters):
    from paper_2102_10245_b200.cpd import DeviceCpAls

    cfg = synth.CONFIGS[5]
    t0 = time.time()
    coords, vals = synth.make_tensor_device(5, nnz=nnz)
    alto = build_alto_device(build_masks(cfg.dims), coords, vals)
    del coords
    torch.cuda.synchronize()
    print(f"gen+build {time.time() - t0:.1f} s, nnz {alto.nnz}", flush=True)
    st = DeviceCpAls(alto, 16, seed=0, backend="atomic", partitions=8)
    m0 = st.mttkrp(0)
    hist = [st.fit(m0, 0)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        hist.append(st.sweep())
    e1.record()
    torch.cuda.synchronize()
    print(f"cfg5 law, {alto.nnz} nnz: CP-ALS {e0.elapsed_time(e1) / iters:.2f} ms/iter over {iters} iters; "
          f"fit {hist}", flush=True)
    print(f"peak memory {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")


if __name__ == "__main__" and sys.argv[1] != "cpals":
    what = sys.argv[1]
    if what == "exact":
        exact(int(sys.argv[2]) if len(sys.argv) > 2 else 50_000_000, len(sys.argv) <= 3)
    else:
        cpals5(int(sys.argv[2]) if len(sys.argv) > 2 else 500_000_000, int(sys.argv[3]) if len(sys.argv) > 3 else 10)


def cpals_breakdown(cfg_id=2, nnz=None, iters=3):
    """CP-ALS sweeps on device (streaming backend) for an ncu launch list."""
    from paper_2102_10245_b200.cpd import DeviceCpAls

    cfg = synth.CONFIGS[cfg_id]
    coords, vals = synth.make_tensor_device(cfg_id, nnz=nnz)
    alto = build_alto_device(build_masks(cfg.dims), coords, vals)
    st = DeviceCpAls(alto, cfg.rank, seed=0, backend="atomic", partitions=8)
    st.sweep()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        st.sweep()
    e1.record()
    torch.cuda.synchronize()
    print(f"{cfg.name}: CP-ALS {e0.elapsed_time(e1) / iters:.2f} ms/iter", flush=True)


if __name__ == "__main__" and sys.argv[1] == "cpals":
    cpals_breakdown(int(sys.argv[2]))
