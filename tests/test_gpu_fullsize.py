"""Full-size parity: every mode of every BASELINE.json config at its stated
nonzero count, device MTTKRP vs the float64 C oracle (oracle/mttkrp_oracle.c,
a bitwise restatement of the reference's mttkrp_oracle, mttkrp.py:64-77,
pinned by tests/test_oracle_c.py) on the same seeded inputs.

Per mode four device paths are checked:
  * `stream`  - the float32 mode-stream kernel the bench times (mttkrp_stream,
                float32 output): relative Frobenius error <= 1e-5 (north star);
  * `pull`    - the K8/K9 pull engine (slice interval buffers + deterministic
                pull, the Buffered scheme) with float32 factors and output:
                <= 1e-5, and bitwise equal across two runs;
  * `alto`    - the single-copy ALTO-order kernel (packed keys + sub-tile
                order, no per-mode stream), float32 output: <= 1e-5 (its
                Zipf-head rows merge once per 128-element sub-tile, 2-4M
                times per head row on cfg5: the per-row copy counts of
                alto_hot_copies bound the float32 merges per copy; the
                uniform 64-copy plan of round 1 measured 1.3-3.4e-5 there);
  * `api`     - the reference-facing default path `mttkrp(tensor, factors,
                mode, partitions=16)` with float64 factors (auto plan =
                Buffered on every mode, SURVEY §7.3 item 7 -> the
                deterministic device engine): <= 1e-10.
Inputs: the BASELINE law drawn on the device (synth.make_tensor_device),
fp32-rounded values and factors (the reference upcasts them exactly,
SURVEY §8.0); the oracle consumes the identical coordinate/value arrays.
Each run appends its errors to gpurun_out/fullsize_parity.jsonl.
"""

import json
import os
import time

import numpy as np
import pytest

from oracle import oracle_c
from paper_2102_10245_b200 import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(1, 100_000), (2, 50_000_000), (3, 100_000_000), (4, 20_000_000), (5, 500_000_000)]


def _record(rec):
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "fullsize_parity.jsonl"), "a") as f:
        f.write(json.dumps(rec) + "\n")


@pytest.mark.parametrize("cfg,nnz", CASES, ids=[f"cfg{c}-{n}nnz" for c, n in CASES])
def test_fullsize_mttkrp_all_modes_vs_oracle(at, cfg, nnz):
    import torch

    from paper_2102_10245_b200.format import build_alto_device
    from paper_2102_10245_b200.layout import build_masks
    from paper_2102_10245_b200.mttkrp import factors_to_device, mttkrp_pull, mttkrp_stream

    c = synth.CONFIGS[cfg]
    assert c.nnz == nnz
    dims, rank = c.dims, c.rank
    fp32 = c.value_dtype == "float32"
    coords, vals = synth.make_tensor_device(cfg)
    alto = build_alto_device(build_masks(dims), coords, vals)
    cols = [coords[:, n].to(torch.int32).cpu().numpy() for n in range(len(dims))]
    vals_h = vals.cpu().numpy()
    del coords, vals
    rng = np.random.default_rng(synth.SEED_FACTOR_BASE + cfg)
    fdt = np.float32 if fp32 else np.float64
    factors = [rng.random((d, rank)).astype(fdt) for d in dims]
    f64 = [f.astype(np.float64) for f in factors]
    fdev = factors_to_device(factors)
    tol_fast = 1e-5 if fp32 else 1e-12
    out_dt = torch.float32 if fp32 else torch.float64
    errs = {}
    for mode in range(len(dims)):
        t0 = time.time()
        ref = oracle_c.mttkrp_coo(cols, vals_h, f64, mode)
        t_oracle = time.time() - t0
        got = {}
        got["stream"] = mttkrp_stream(alto, fdev, mode, out_dtype=out_dt).cpu().numpy()
        p = mttkrp_pull(alto, fdev, mode, out_dtype=out_dt)
        if p is not None:
            # the Buffered engine is bitwise reproducible at full size
            assert torch.equal(p, mttkrp_pull(alto, fdev, mode, out_dtype=out_dt)), (cfg, mode)
            got["pull"] = p.cpu().numpy()
        if rank in (16, 32) and max(build_masks(dims).bits) <= 31:
            got["alto"] = mttkrp_stream(alto, fdev, mode, out_dtype=out_dt, planned="pos").cpu().numpy()
        got["api"] = at.mttkrp(alto, f64, mode, partitions=16)
        e = {k: oracle_c.rel_error(v, ref) for k, v in got.items()}
        errs[mode] = e
        _record({"cfg": cfg, "nnz": nnz, "mode": mode, "rank": rank, "rel_err": e, "oracle_s": t_oracle,
                 "oracle_threads": oracle_c.host_threads()})
        del got, ref
        alto._cache.clear()  # per-mode plans: keep the HBM working set to one mode
        torch.cuda.empty_cache()
    for mode, e in errs.items():
        assert e["stream"] <= tol_fast, (cfg, nnz, mode, e)
        if "alto" in e:
            assert e["alto"] <= tol_fast, (cfg, nnz, mode, e)
        if "pull" in e:
            assert e["pull"] <= tol_fast, (cfg, nnz, mode, e)
        assert e["api"] <= (1e-10 if fp32 else 1e-12), (cfg, nnz, mode, e)
    del alto, fdev
    torch.cuda.empty_cache()
