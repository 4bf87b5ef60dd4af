"""Simulated key-range sharding of a BASELINE config on one GPU:
per G in {2, 4, 8} and per cut rule (equal-nnz = the API partition,
cost-balanced = dist.build_shard's model), the per-shard nonzeros, the
modelled cost share, rows touched per mode, rows shared by >= 2 shards, and
the owner-directed exchange volume per rank per ALS sweep (both legs, all
modes) next to what an all-reduce of the global shared-row set would move.
  python tools/sim_shards.py [cfg] -> one JSON line per (G, cut)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10245_b200 import synth  # noqa: E402
from paper_2102_10245_b200.format import build_alto_device  # noqa: E402
from paper_2102_10245_b200.layout import build_masks, delinearize_device  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    c = synth.CONFIGS[cfg]
    R, S = c.rank, 4
    coords, vals = synth.make_tensor_device(cfg)
    lay = build_masks(c.dims)
    alto = build_alto_device(lay, coords, vals)
    del coords
    torch.cuda.empty_cache()
    m = alto.nnz
    kv = 8 * lay.n_words + 4
    rows = [delinearize_device(lay, alto.keys, n).to(torch.int32) for n in range(len(c.dims))]
    w = torch.full((m,), float(kv), dtype=torch.float64, device="cuda")
    for n, d in enumerate(c.dims):
        cnt = torch.bincount(rows[n].long(), minlength=d).to(torch.float64)
        w += R * S / cnt[rows[n].long()]
    cw = torch.cumsum(w, 0)
    total = float(cw[-1].item())
    for G in (2, 4, 8):
        for cut in ("equal_nnz", "cost_balanced"):
            if cut == "equal_nnz":
                q, r = divmod(m, G)
                b = [0]
                for g in range(G):
                    b.append(b[-1] + q + (1 if g < r else 0))
            else:
                b = [0] + [int(torch.searchsorted(cw, torch.tensor(total * g / G, dtype=torch.float64,
                                                                      device="cuda")).item()) for g in range(1, G)] + [m]
            cost = [(float(cw[b[g + 1] - 1].item()) - (float(cw[b[g] - 1].item()) if b[g] else 0.0)) / total
                    for g in range(G)]
            per_rank_bytes = [0] * G
            allreduce_rows = 0
            touched_rows = []
            shared_rows = []
            for n, d in enumerate(c.dims):
                tch = torch.zeros((G, d), dtype=torch.bool, device="cuda")
                for g in range(G):
                    tch[g, rows[n][b[g]:b[g + 1]].long()] = True
                cnt = tch.sum(0)
                shared = cnt >= 2
                first = torch.argmax(tch.to(torch.int8), 0)
                touched_rows.append([int(tch[g].sum().item()) for g in range(G)])
                shared_rows.append(int(shared.sum().item()))
                allreduce_rows += int(shared.sum().item())
                for g in range(G):
                    send = int((tch[g] & shared & (first != g)).sum().item())
                    recv = int((shared & (first == g)).to(torch.int64).mul(cnt - 1).sum().item())
                    per_rank_bytes[g] += 2 * (send + recv) * R * S
                del tch
            print(json.dumps({"cfg": cfg, "G": G, "cut": cut, "nnz": [b[g + 1] - b[g] for g in range(G)],
                              "cost_share": cost, "rows_touched": touched_rows, "rows_shared": shared_rows,
                              "owner_directed_bytes_per_rank_per_sweep": per_rank_bytes,
                              "max_rank_bytes": max(per_rank_bytes),
                              "ring_allreduce_bytes_per_rank_per_sweep": 2 * (G - 1) / G * allreduce_rows * R * S}),
                  flush=True)


if __name__ == "__main__":
    main()
