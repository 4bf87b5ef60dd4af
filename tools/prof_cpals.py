"""Per-phase CUDA-event timing of one CP-ALS sweep on a BASELINE config (ad-hoc):
  python tools/prof_cpals.py [cfg] [nnz]"""
import sys
import time

import torch

from paper_2102_10245_b200 import synth
from paper_2102_10245_b200.cpd import DeviceCpAls
from paper_2102_10245_b200.format import build_alto_device
from paper_2102_10245_b200.layout import build_masks


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    nnz = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else None
    c = synth.CONFIGS[cfg]
    coords, vals = synth.make_tensor_device(cfg, nnz=nnz)
    alto = build_alto_device(build_masks(c.dims), coords, vals)
    del coords, vals
    st = DeviceCpAls(alto, c.rank, seed=0, backend="atomic", partitions=8)
    st.sweep()
    torch.cuda.synchronize()
    for it in range(2):
        times = {}
        for mode in range(len(c.dims)):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            st.backend.run(st.gather_factors(), mode, allow_f32=True)
            ev[1].record()
            st.update(mode)
            ev[2].record()
            torch.cuda.synchronize()
            times[mode] = [round(ev[0].elapsed_time(ev[1]), 3), round(ev[1].elapsed_time(ev[2]), 3)]
        t0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.sweep()
        e1.record()
        torch.cuda.synchronize()
        print(f"cfg{cfg} nnz {alto.nnz}: per mode [mttkrp alone, full update incl. mttkrp] ms {times}; "
              f"sweep {e0.elapsed_time(e1):.2f} ms (wall {1e3 * (time.time() - t0):.1f})", flush=True)


if __name__ == "__main__":
    main()
