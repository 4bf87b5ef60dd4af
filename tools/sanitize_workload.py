"""Small workload touching every device entry point of the hot path, for
compute-sanitizer (memcheck / racecheck / synccheck) runs:
  compute-sanitizer --tool memcheck python tools/sanitize_workload.py"""
import importlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_10245_b200 as at  # noqa: E402
from paper_2102_10245_b200 import synth  # noqa: E402

mk = importlib.import_module("paper_2102_10245_b200.mttkrp")


def main():
    for cfg, nnz in ((1, 100_000), (5, 60_000), (4, 50_000)):
        st = synth.make_tensor(cfg, nnz=nnz)
        dims = st.config.dims
        coo = at.CooTensor(dims, st.coords, st.values.astype(np.float64))
        for dt in ("float64", "float32"):
            alto = at.build_alto(coo, dtype=dt)
            parts = at.partition(alto, 8)
            rng = np.random.default_rng(1)
            fac = [rng.random((d, 16)) for d in dims]
            for mode in range(len(dims)):
                at.mttkrp_oracle(coo, fac, mode)
                for strat in (at.Strategy.BUFFERED, at.Strategy.ATOMIC):
                    plan = at.plan_conflicts(alto, parts, mode, force_strategy=strat)
                    t = at.apply_boundary_flags(alto, plan) if plan.flag_bit is not None else alto
                    at.mttkrp_par(t, parts, plan, fac, mode)
                f32 = mk.factors_to_device([f.astype(np.float32) for f in fac])
                if dt == "float32":
                    mk.mttkrp_stream(alto, f32, mode, out_dtype=torch.float32)
                    mk.mttkrp_pull(alto, f32, mode, out_dtype=torch.float32)
                    mk.mttkrp_stream(alto, f32, mode, out_dtype=torch.float32, planned="pos")
                mk.mttkrp_exact(alto, mk.factors_to_device(fac), mode)
            at.cpd_als(alto, 16, max_iters=2, tol=0.0, backend="auto", partitions=4)
            at.cpd_als(alto, 16, max_iters=2, tol=0.0, backend="atomic", partitions=4)
            at.cpd_als(alto, 5, max_iters=2, tol=0.0, backend="seq")
            at.deserialize(at.serialize(alto))
        dup = np.concatenate([st.coords, st.coords[::5]])
        at.CooTensor(dims, dup, np.ones(dup.shape[0])).coalesce()
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
