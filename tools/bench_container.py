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


if __name__ == "__main__":
    main()
