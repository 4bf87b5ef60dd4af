"""How much of a config's factor-row traffic could any L2-sized cache keep?
For every mode: the share of element references that go to its K most
referenced rows, K * rank * 4 bytes = 16/32/64/96 MB (an ideal static cache
of that size), next to the rows referenced at all.  python tools/reuse_stats.py [cfg]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_10245_b200 import synth  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    c = synth.CONFIGS[cfg]
    coords, _ = synth.make_tensor_device(cfg)
    rowb = c.rank * 4
    for n, d in enumerate(c.dims):
        cnt = torch.bincount(coords[:, n], minlength=d)
        srt, _ = torch.sort(cnt, descending=True)
        cum = torch.cumsum(srt, 0).double() / coords.shape[0]
        res = {"cfg": cfg, "mode": n, "rows": d, "rows_referenced": int((cnt > 0).sum().item()),
               "factor_MB": d * rowb / 1e6, "max_row_count": int(srt[0].item()), "share_of_references_in_top_rows": {}}
        for mb in (16, 32, 64, 96):
            k = min(d, mb * (1 << 20) // rowb)
            res["share_of_references_in_top_rows"][f"{mb}MB"] = round(float(cum[k - 1].item()), 4)
        print(json.dumps(res), flush=True)
        del cnt, srt, cum


if __name__ == "__main__":
    main()
