"""Summarise ncu outputs brought back from the GPU box into profiles/.

  python profiles/summarize.py launches <launches.csv> <out.md>
  python profiles/summarize.py full <report.ncu-rep> <out.json>

`launches`: per-kernel totals of gpu__time_duration.sum from the
--metrics launch-list pass (cold-cache, serialised: compare SHARES).
`full`: the headline metrics of each profiled launch of a --set full capture
(duration, DRAM bytes, L2 hit rate, L1/LTS throughput, warp stalls).
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys


STEP_KERNELS = ("mstream_kernel<", "mstream_blk_kernel<", "hot_reduce_rows_kernel<float>", "krp_pair_kernel")


def launches(path: str, out: str) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        name = r[4].split("(")[0]
        tot[name] += float(r[14]) / 1e3  # ns -> us
        cnt[name] += 1
    grand = sum(tot.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{name}` | {cnt[name]} | {t:.1f} | {t / grand * 100:.1f}% |")
    step = {n: t for n, t in tot.items() if any(k in n for k in STEP_KERNELS)}
    st = sum(step.values()) or 1.0
    lines += ["", "Kernels of the timed bench step (f32 output; the process above also "
              "generates inputs, builds the tensor and runs the e2e/fp64 API leg):", "",
              "| kernel | share of step |", "|---|---|"]
    for name, t in sorted(step.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{name}` | {t / st * 100:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "lts__t_sectors_srcunit_tex_op_red.sum", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg",
    "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum",
    "sm__cycles_elapsed.avg", "launch__registers_per_thread", "launch__grid_size", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]


def full(path: str, out: str) -> None:
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:160]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = {"value": r[i], "unit": units[i]}
        stalls = {h.split("stalled_")[1]: float(v or 0) for h, v in zip(hdr, r)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        d["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:4000])


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
