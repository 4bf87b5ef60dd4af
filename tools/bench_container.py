"""`.alto` container streaming throughput on a BASELINE config (ad-hoc):
  python tools/bench_container.py [cfg] [nnz]
Builds the tensor on the device, writes it with write_alto, reads it back
with read_alto (disk/page cache -> pinned buffers -> HBM) and checks the
round trip; prints sizes and GB/s against rebuilding (build_alto_device)."""
import os
import sys
import tempfile
import time

import torch

import paper_2102_10245_b200 as at
from paper_2102_10245_b200 import synth
from paper_2102_10245_b200.format import build_alto_device
from paper_2102_10245_b200.layout import build_masks


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    nnz = int(sys.argv[2]) if len(sys.argv) > 2 else None
    c = synth.CONFIGS[cfg]
    coords, vals = synth.make_tensor_device(cfg, nnz=nnz)
    torch.cuda.synchronize()
    t0 = time.time()
    alto = build_alto_device(build_masks(c.dims), coords, vals)
    torch.cuda.synchronize()
    t_build = time.time() - t0
    path = os.path.join(tempfile.gettempdir(), f"bench_cfg{cfg}.alto")
    t0 = time.time()
    at.write_alto(alto, path)
    t_write = time.time() - t0
    size = os.path.getsize(path)
    t0 = time.time()
    back = at.read_alto(path, dtype="float32")
    torch.cuda.synchronize()
    t_read = time.time() - t0
    ok = torch.equal(back.keys, alto.keys) and torch.equal(back.vals, alto.vals)
    os.remove(path)
    print(f"cfg{cfg}: nnz {alto.nnz}, file {size / 1e9:.2f} GB; write_alto {t_write:.2f} s "
          f"({size / t_write / 1e9:.2f} GB/s), read_alto {t_read:.2f} s ({size / t_read / 1e9:.2f} GB/s), "
          f"device rebuild from coordinates {t_build * 1e3:.0f} ms; round trip equal: {ok}", flush=True)


def coalesce_bench(m=50_000_000):
    """Device coalesce of m uniformly drawn rows vs the oracle
    restatement of the reference (numpy lexsort + bincount) on a 2M sample."""
    import numpy as np

    from oracle import alto_oracle as orc
    from paper_2102_10245_b200.coo import coalesce_device

    dims = (1000, 800, 600)  # random_tensor-style draw: ~5 % collisions
    rng = np.random.default_rng(5)
    c = rng.integers(0, dims, size=(m, 3), dtype=np.int64)
    v = rng.random(m)
    cd = torch.from_numpy(c).cuda()
    vd = torch.from_numpy(v).cuda()
    coalesce_device(dims, cd, vd)
    torch.cuda.synchronize()
    t0 = time.time()
    oc, ov = coalesce_device(dims, cd, vd)
    torch.cuda.synchronize()
    t_dev = time.time() - t0
    s = 2_000_000
    t0 = time.time()
    orc.coalesce(c[:s], v[:s])
    t_cpu = time.time() - t0
    print(f"coalesce: {m} rows -> {oc.shape[0]} distinct in {t_dev * 1e3:.1f} ms on the device "
          f"({m / t_dev / 1e9:.2f} G rows/s); reference algorithm (numpy, 1 core) {s / t_cpu / 1e6:.1f} M rows/s "
          f"on a {s}-row sample", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "coalesce":
        coalesce_bench()
    else:
        main()
