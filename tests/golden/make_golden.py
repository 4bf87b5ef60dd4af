"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the unmodified reference package from /root/reference/pkg/src and
records its outputs on seeded inputs into tests/golden/*.npz.  The fixtures
travel with the repo; the GPU box never needs /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import altotensor as at  # noqa: E402  (the reference)
from altotensor.cpd import cpd_als  # noqa: E402
from altotensor.format import Strategy  # noqa: E402
from altotensor.mttkrp import mttkrp_oracle, mttkrp_par, mttkrp_seq  # noqa: E402

from paper_2102_10245_b200 import synth  # noqa: E402  (seeded generator only)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case_record(name, coo, counts, rank, fseed, store_inputs=True, cpd_iters=None, cpd_rank=None,
                cpd_seed=0, backends=("seq",), with_mttkrp=True, project=False):
    rec: dict = {}
    proj_u = np.random.default_rng(99).random(rank)

    def put_out(key, arr):
        # large outputs are stored as a projection onto a seeded vector + norm
        if project:
            rec[key + "_proj"] = arr @ proj_u
            rec[key + "_fro"] = np.asarray(np.linalg.norm(arr))
        else:
            rec[key] = arr

    meta: dict = {"name": name, "dims": list(coo.dims), "nnz": int(coo.nnz), "rank": rank, "fseed": fseed,
                  "counts": list(counts)}
    alto = at.build_alto(coo)
    lay = alto.layout
    meta.update(bits=list(lay.bits), positions=[list(p) for p in lay.positions],
                masks=[str(m) for m in lay.masks], total_bits=lay.total_bits, width=lay.width)
    meta["coords_sha"] = sha(coo.coords)
    meta["values_sha"] = sha(coo.values)
    meta["indices_sha"] = sha(alto.indices)
    meta["sorted_values_sha"] = sha(alto.values)
    if store_inputs:
        rec["coords"] = coo.coords
        rec["values"] = coo.values
        rec["indices"] = alto.indices
        rec["sorted_values"] = alto.values
    meta["with_mttkrp"] = with_mttkrp
    meta["project"] = project
    rng = np.random.default_rng(fseed)
    factors = [rng.random((d, rank)) for d in coo.dims] if with_mttkrp else None
    if store_inputs and with_mttkrp:
        for n, f in enumerate(factors):
            rec[f"factor_{n}"] = f
    plans = {}
    for count in counts:
        parts = at.partition(alto, count)
        rec[f"L{count}_offsets"] = parts.offsets
        rec[f"L{count}_intervals"] = parts.intervals
        meta[f"L{count}_spans"] = [[str(a), str(b)] for a, b in parts.spans]
        for mode in range(lay.order):
            for force in (None, Strategy.ATOMIC, Strategy.BUFFERED):
                plan = at.plan_conflicts(alto, parts, mode, force_strategy=force)
                key = f"L{count}_m{mode}_{'auto' if force is None else force.value}"
                plans[key] = {
                    "strategy": plan.strategy.value,
                    "reuse": plan.reuse,
                    "overlaps": None if plan.overlaps is None else [[list(r) for r in o] for o in plan.overlaps],
                    "flag_bit": plan.flag_bit,
                }
                if force is Strategy.ATOMIC:
                    if plan.flag_bit is not None:
                        flagged = at.apply_boundary_flags(alto, plan)
                        meta[key + "_flagged_sha"] = sha(flagged.indices)
                        if store_inputs:
                            rec[key + "_flagged"] = flagged.indices
                        run = flagged
                    else:
                        run = alto
                    if with_mttkrp:
                        put_out(key + "_mttkrp", mttkrp_par(run, parts, plan, factors, mode, workers=4))
                if force is Strategy.BUFFERED and with_mttkrp:
                    put_out(key + "_mttkrp", mttkrp_par(alto, parts, plan, factors, mode, workers=4))
    meta["plans"] = plans
    for mode in range(lay.order if with_mttkrp else 0):
        put_out(f"m{mode}_oracle", mttkrp_oracle(coo, factors, mode))
        put_out(f"m{mode}_seq", mttkrp_seq(alto, factors, mode))
    if cpd_iters is not None:
        for be in backends:
            model = cpd_als(alto, rank=cpd_rank or rank, max_iters=cpd_iters, tol=0.0, seed=cpd_seed, backend=be,
                            workers=4, partitions=4)
            rec[f"cpd_{be}_fit"] = np.asarray(model.fit_history)
            rec[f"cpd_{be}_weights"] = model.weights
            if store_inputs:
                for n, f in enumerate(model.factors):
                    rec[f"cpd_{be}_factor_{n}"] = f
        meta["cpd"] = {"iters": cpd_iters, "rank": cpd_rank or rank, "seed": cpd_seed, "backends": list(backends)}
    rec["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **rec)
    print(f"wrote {name}.npz  nnz={coo.nnz} width={lay.width}")


def main():
    # 1. the paper's worked example (pkg/tests/conftest.py:8-20)
    coords = np.array([[1, 0, 0], [3, 0, 1], [0, 3, 0], [2, 2, 1], [3, 2, 0], [1, 6, 1]])
    ex = at.CooTensor((4, 8, 2), coords, np.arange(1.0, 7.0))
    case_record("worked_example", ex, [1, 2, 3, 6], rank=2, fseed=5, cpd_iters=3, cpd_rank=2, cpd_seed=0)
    # 2. seeded random tensors in the reference's own test shapes
    case_record("r3_25x30x18", at.random_tensor((25, 30, 18), 2500, seed=10), [1, 4, 6, 8], rank=8, fseed=11,
                cpd_iters=4, cpd_rank=3, cpd_seed=17, backends=("seq", "buffered", "atomic", "oracle"))
    case_record("r4_12x9x7x11", at.random_tensor((12, 9, 7, 11), 1500, seed=12), [1, 3, 5], rank=5, fseed=13)
    case_record("r5_8x9x7x6x5", at.random_tensor((8, 9, 7, 6, 5), 900, seed=21), [1, 7], rank=16, fseed=22)
    case_record("skew_4x100x4", at.random_tensor((4, 100, 4), 64, seed=14), [1, 2, 64], rank=2, fseed=15)
    # 128-bit keys (pkg/tests/test_format.py:38-48 shape)
    rng = np.random.default_rng(9)
    dims = (1 << 40, 1 << 30, 1 << 40)
    wc = np.unique(rng.integers(0, dims, size=(300, 3), dtype=np.int64), axis=0)
    case_record("wide_128", at.CooTensor(dims, wc, rng.random(len(wc))), [1, 4], rank=4, fseed=3, with_mttkrp=False)
    # no free flag bit: total_bits == width (pkg/tests/test_format.py:136-142)
    full = at.CooTensor((1 << 32, 1 << 32), [[0, 0], [5, 9], [7, 1], [1 << 31, 3]], [1.0, 2.0, 3.0, 4.0])
    case_record("full_width_64", full, [1, 2], rank=3, fseed=4, with_mttkrp=False)
    # 128-bit keys with materialisable factors: 71-bit layout like cfg5 at toy extents
    rng = np.random.default_rng(31)
    dims = (40_000_000, 20_000_000, 1_000_000)
    wc = np.unique(rng.integers(0, (64, 64, 64), size=(3000, 3), dtype=np.int64), axis=0)
    case_record("wide_cfg5_layout", at.CooTensor(dims, wc, rng.random(len(wc))), [1, 5], rank=4, fseed=6,
                with_mttkrp=False)
    # 3. BASELINE cfg1 at full size (synthetic generator, seeded): outputs only
    st = synth.make_tensor(1)
    coo = at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64))
    case_record("cfg1", coo, [8], rank=16, fseed=synth.SEED_FACTOR_BASE + 1, store_inputs=False, cpd_iters=5,
                cpd_rank=16, cpd_seed=0)
    # 4. cfg2 law at reduced size (fp32-rounded values), outputs only
    st = synth.make_tensor(2, nnz=200_000)
    coo = at.CooTensor(st.config.dims, st.coords, st.values.astype(np.float64))
    case_record("cfg2_200k", coo, [8], rank=16, fseed=synth.SEED_FACTOR_BASE + 2, store_inputs=False,
                project=True)


if __name__ == "__main__":
    main()
