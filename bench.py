"""ALTO MTTKRP benchmark on B200 (driver contract: one JSON line from rank 0).

Workload (BASELINE.json configs[1], "cfg2"): 3-mode 200,000 x 150,000 x
100,000 tensor, 50M distinct nonzeros, Zipf(1.1) per mode, fp32 values,
rank-16 fp32 factors; one step = MTTKRP over all 3 modes (streaming kernel).
Metric: MTTKRP nonzeros/s (mode-averaged: 3*nnz per step / step time).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 (torchrun): nonzeros are sharded by linearized-key range (ALTO
partitions), factors replicated; each mode's step adds the shared-row
exchange of dist.py (rows touched by >= 2 shards packed into one NCCL
all-reduce), timed as the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def bytes_alg(dims, nnz, key_bytes, val_bytes, rank, fbytes, mode):
    """M(K+V) + sum_{m!=n} I_m R S + I_n R S."""
    return nnz * (key_bytes + val_bytes) + sum(d * rank * fbytes for d in dims)


def cpu_baseline_sample(cfg_id: int, sample_nnz: int, threads: int, reps: int = 3):
    """The reference's CPU MTTKRP (installed reference when present, else the
    oracle port of Buffered mttkrp_par) on a bounded same-law sample, all modes."""
    from paper_2102_10245_b200 import synth

    c = synth.CONFIGS[cfg_id]
    step, kind, what = reference_step(cfg_id, sample_nnz, threads)
    times = []
    for _rep in range(reps + 1):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    t = sum(times[1:]) / reps  # first rep is warm-up (cli.py:198-203 protocol)
    return {"value": len(c.dims) * sample_nnz / t, "unit": "nnz/s", "cores": threads, "kind": kind,
            "sample": f"{sample_nnz} nnz drawn from the {c.name} law (same dims, {laws_str(c)}, {c.value_dtype} values), "
                      f"all {len(c.dims)} modes, {what}, mean of {reps} after 1 warm-up",
            "seconds_per_step": t}


def _load_installed_reference():
    """The unmodified reference package installed into baseline/_ref (see
    DESIGN.md §8), or None when that install is absent."""
    ref_dir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "altotensor")):
        return None
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    import altotensor

    return altotensor


def reference_step(cfg_id: int, sample: int, threads: int):
    """One all-modes MTTKRP pass of the reference on a bounded same-law sample:
    the installed unmodified reference when present, else the oracle port.
    Returns (step, kind, description)."""
    from paper_2102_10245_b200 import synth

    st = synth.make_tensor(cfg_id, nnz=sample)
    c = st.config
    rng = np.random.default_rng(synth.SEED_FACTOR_BASE + cfg_id)
    factors = [rng.random((d, c.rank)).astype(np.float32).astype(np.float64) for d in c.dims]
    at = _load_installed_reference()
    if at is not None:
        # The reference's own public API and stock path, prepared as its CLI
        # does (cli.py `_prepare`: partition, plan, flags outside the timed
        # loop), then mttkrp_par per mode with every host thread.
        tensor = at.build_alto(at.CooTensor(c.dims, st.coords, st.values.astype(np.float64)))
        parts = at.partition(tensor, threads)
        prepared = []
        for mode in range(len(c.dims)):
            plan = at.plan_conflicts(tensor, parts, mode)
            t_m = at.apply_boundary_flags(tensor, plan) if (
                plan.strategy is at.Strategy.ATOMIC and plan.flag_bit is not None) else tensor
            prepared.append((t_m, plan))

        def step():
            for mode, (t_m, plan) in enumerate(prepared):
                at.mttkrp_par(t_m, parts, plan, factors, mode, threads)

        kind = "reference"
        what = (f"unmodified reference altotensor {at.__version__} (baseline/_ref), mttkrp_par per mode "
                f"with the auto conflict plan, {threads} partitions/workers")
    else:
        from oracle import alto_oracle as orc

        lay = orc.build_layout(c.dims)
        words, vals = orc.build(lay, st.coords, st.values.astype(np.float64))
        offs, iv, _ = orc.partition(lay, words, threads)

        def step():
            for mode in range(len(c.dims)):
                orc.mttkrp_buffered(lay, words, vals, factors, mode, offs, iv, workers=threads)

        kind = "port"
        what = f"oracle port of the reference mttkrp_par (Buffered, {threads} workers); baseline/_ref not installed"

    return step, kind, what


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    sample = args.cpu_sample
    step, kind, what = reference_step(args.config, sample, threads)
    from paper_2102_10245_b200 import synth

    c = synth.CONFIGS[args.config]
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    t = (time.perf_counter() - t0) / args.steps
    value = len(c.dims) * sample / t
    line = {
        "impl": "reference", "metric": "MTTKRP nonzeros/sec (mode-averaged)", "value": value, "unit": "nnz/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json law)",
        "config": {"workload": f"{c.name}: dims {list(c.dims)}, {laws_str(c)}, rank {c.rank}; CPU sample {sample} nnz",
                   "sample_nnz": sample, "threads": threads},
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads, "kind": kind,
                         "sample": f"{sample} nnz of the {c.name} law, all modes, {what}"},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def laws_str(c) -> str:
    """Coordinate laws of a synthetic config, e.g. 'modes: zipf(1.1), zipf(1.1), zipf(1.1)'."""
    return "modes: " + ", ".join(f"zipf({s})" if law == "zipf" else "uniform" for law, s in c.laws)


def traffic_from_profile(cfg_id: int):
    """Per-launch DRAM bytes (read + write) of the dominant kernel, averaged
    over the captured launches of the latest committed `ncu --set full`
    capture of this workload (profiles/r*_cfg<id>_mstream_ncu.json)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_cfg{cfg_id}_mstream_ncu.json")))
    if not files:
        return None, None
    try:
        rows = json.load(open(files[-1]))
        vals = []
        for r in rows:
            if "mstream_kernel" in r["kernel"] or "mstream_blk_kernel" in r["kernel"]:
                rd = float(r["dram__bytes_read.sum"]["value"])
                wr = float(r["dram__bytes_write.sum"]["value"])
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                vals.append(rd * scale[r["dram__bytes_read.sum"]["unit"]] +
                            wr * scale[r["dram__bytes_write.sum"]["unit"]])
        return (sum(vals) / len(vals) if vals else None), os.path.relpath(files[-1], ROOT)
    except Exception:
        return None, None


def flush_l2(buf):
    buf.add_(1.0)


def _events(n):
    import torch

    return [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]


def cache_bytes(alto, keys) -> int:
    """HBM bytes held by the tensor's cached plans whose cache key starts with one of `keys`."""
    import torch

    tot = 0

    def walk(v):
        nonlocal tot
        if isinstance(v, torch.Tensor):
            tot += v.numel() * v.element_size()
        elif isinstance(v, (tuple, list)):
            for x in v:
                walk(x)
        elif isinstance(v, dict):
            for x in v.values():
                walk(x)

    for k, v in alto._cache.items():
        name = k[0] if isinstance(k, tuple) else k
        if name in keys:
            walk(v)
    return tot


def time_modes(fn, N, steps, l2, stream):
    """Per-mode CUDA-event times (ms) of fn(mode), L2 flushed before each
    all-modes step; returns (step_ms list, per-mode mean ms)."""
    import torch

    step_ev = _events(steps)
    mode_ev = [_events(N) for _ in range(steps)]
    for k in range(steps):
        flush_l2(l2)
        step_ev[k][0].record(stream)
        for n in range(N):
            mode_ev[k][n][0].record(stream)
            fn(n)
            mode_ev[k][n][1].record(stream)
        step_ev[k][1].record(stream)
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    mode_ms = [sum(mode_ev[k][n][0].elapsed_time(mode_ev[k][n][1]) for k in range(steps)) / steps for n in range(N)]
    return step_ms, mode_ms


def timed_once(fn, stream):
    import torch

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def run_b200(args):
    import importlib

    import torch
    import torch.distributed as dist

    import paper_2102_10245_b200 as at
    from paper_2102_10245_b200 import synth
    from paper_2102_10245_b200.format import AltoTensor, build_alto_device
    from paper_2102_10245_b200.layout import build_masks

    mk = importlib.import_module("paper_2102_10245_b200.mttkrp")
    if getattr(args, "l2_hot_mb", None) is not None:
        mk.MS_L2_HOT_MB = args.l2_hot_mb
    ws, rank, local = dist_env()
    # functional check of the multi-rank path on a one-GPU box only
    # (ALTO_BENCH_TEST_GLOO=1: every rank on cuda:0, gloo collectives; numbers
    # from such a run are not measurements)
    test_gloo = os.environ.get("ALTO_BENCH_TEST_GLOO") == "1"
    if test_gloo:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if test_gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = synth.CONFIGS[args.config]
    nnz_total = args.nnz or cfg.nnz
    t_gen = time.time()
    vdt = torch.float32 if cfg.value_dtype == "float32" else torch.float64
    if args.gen == "host":
        st = synth.make_tensor(args.config, nnz=nnz_total)
        coords = torch.from_numpy(st.coords).to(dev)
        vals = torch.from_numpy(st.values).to(device=dev, dtype=vdt)
    else:
        coords, vals = synth.make_tensor_device(args.config, nnz=nnz_total, device=dev)
    torch.cuda.synchronize()
    t_gen = time.time() - t_gen
    dims = cfg.dims
    R = args.rank or cfg.rank
    N = len(dims)
    lay = build_masks(dims)
    stream = torch.cuda.current_stream()
    exch_bytes = 0
    shard_info = None
    if ws > 1:
        from paper_2102_10245_b200.dist import build_shard

        e0 = time.time()
        alto, shard_info = build_shard(lay, coords, vals, rank, ws, R)
        torch.cuda.synchronize()
        build_ms = (time.time() - e0) * 1e3
    else:
        build_ms = timed_once(lambda: None, stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        alto = build_alto_device(lay, coords, vals)
        e1.record(stream)
        torch.cuda.synchronize()
        build_ms = e0.elapsed_time(e1)
    del coords, vals
    M = alto.nnz
    fdt = np.float32 if cfg.value_dtype == "float32" else np.float64
    rng = np.random.default_rng(synth.SEED_FACTOR_BASE + args.config)
    factors_host = [rng.random((d, R)).astype(fdt) for d in dims]
    fdev = mk.factors_to_device(factors_host)
    if args.out is None:
        args.out = "f32" if vdt == torch.float32 else "f64"
    odt = torch.float32 if args.out == "f32" else torch.float64
    outs = [torch.empty((d, R), dtype=odt, device=dev) for d in dims]
    l2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    kb, vb, fb = 8 * lay.n_words, 4 if vdt == torch.float32 else 8, np.dtype(fdt).itemsize
    peak, peak_kind = measured_peaks()
    xplans = None
    if ws > 1:
        # shared-row exchange plan per mode (dist.py): only rows touched by
        # >= 2 key-range shards cross NVLink (owner-directed reduce + return)
        from paper_2102_10245_b200.dist import DeviceOps, ShardRows, exchange_shared

        xops = DeviceOps(alto, R)
        xplans = [ShardRows(xops.touched_rows(n)) for n in range(N)]
        exch_bytes = sum(p.n_shared for p in xplans) * R * (4 if args.out == "f32" else 8)

    # ---- one-time per-mode plans (timed; excluded from the per-step time like
    # the reference's partition/plan prep, cli.py:194) ---------------------
    def plan_leg(build, keys):
        for k in [k for k in alto._cache if (k[0] if isinstance(k, tuple) else k) in keys]:
            del alto._cache[k]
        torch.cuda.empty_cache()
        ms = timed_once(build, stream)
        return {"plan_build_ms": ms, "plan_bytes": cache_bytes(alto, keys)}

    def build_ms_plans():
        for n in range(N):
            mk.mttkrp_stream(alto, fdev, n, out=outs[n], hot=not args.no_hot)

    def build_pull_plans():
        for n in range(N):
            mk.pull_stream(alto, n)
            mk.pull_plan(alto, n)

    def build_alto_plans():
        for n in range(N):
            mk.packed_keys(alto)
            mk.subtile_order(alto, n)

    # load every plan/MTTKRP kernel once on a small slice of the tensor
    # (CUDA lazy module loading would otherwise land in the first timed plan build)
    small = AltoTensor(lay, alto.keys[: min(M, 1 << 20)].clone(), alto.vals[: min(M, 1 << 20)].clone())
    for n in range(N):
        mk.mttkrp_stream(small, fdev, n, out=outs[n], hot=not args.no_hot)
        if ws == 1 and not args.skip_paths:
            mk.mttkrp_pull(small, fdev, n, out=outs[n])
            mk.mttkrp_pull(small, fdev, n, out=outs[n], atomic=True)
            if R in (16, 32) and max(lay.bits) <= 31:
                mk.mttkrp_stream(small, fdev, n, out=outs[n], planned="pos")
    del small
    torch.cuda.synchronize()
    ms_keys = ("mstream", "hotms", "hotslots", "row_index", "row_ptr", "packed")
    plans = {"mode_stream": plan_leg(build_ms_plans, ms_keys)}

    def step_stream(n):
        mk.mttkrp_stream(alto, fdev, n, out=outs[n], hot=not args.no_hot)
        if ws > 1:
            exchange_shared(outs[n], xplans[n], xops)

    for _ in range(max(args.warmup, 3)):
        for n in range(N):
            step_stream(n)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        step_ms, mode_ms = time_modes(step_stream, N, args.steps, l2, stream)
    if ws > 1:
        dist.barrier()
    ms = sum(step_ms) / len(step_ms)
    t_ms = torch.tensor([ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms_max = float(t_ms.item())
    value = N * nnz_total / (ms_max * 1e-3)

    per_mode = []
    for n in range(N):
        ba = bytes_alg(dims, M, kb, vb, R, fb, n)
        per_mode.append({"mode": n, "kernel_ms": mode_ms[n], "bytes_alg": ba,
                         "achieved_gbs": ba / (mode_ms[n] * 1e-3) / 1e9, "nnz_per_s": M / (mode_ms[n] * 1e-3)})
    tot_b = sum(p["bytes_alg"] for p in per_mode)
    achieved = tot_b / (sum(mode_ms) * 1e-3) / 1e9
    ms_used = all(any(k[0] == "mstream" and k[1] == n and v for k, v in alto._cache.items() if isinstance(k, tuple))
                  for n in range(N))
    blocked = ms_used and alto.vals.dtype == torch.float32 and mk.MS_RR == 2 and (R == 32 or N >= 4)
    kernel_name = (("alto::mstream_blk_kernel (alto_mstream.cuh)" if blocked else "alto::mstream_kernel (alto_mstream.cuh)")
                   if ms_used else "alto::planned_kernel (alto_fast.cuh)")
    # row gathers per element and mode: N-1 inputs, one fewer per paired input mode
    gathers_per_element = [N - 1 - (len(mk.ms_pairs(dims, n, R, 4)) if ms_used and alto.vals.dtype == torch.float32
                                    else 0) for n in range(N)]
    launches_per_step = 0
    for n in range(N):
        launches_per_step += 1
        if ms_used and alto.vals.dtype == torch.float32:
            launches_per_step += len(mk.ms_pairs(dims, n, R, 4))
        if not args.no_hot:
            hp = (alto._cache.get(("hotms", n, R, odt, mk.ms_tile(alto), mk.MS_ORDER)) if ms_used
                  else alto._cache.get(("hotms", n, R, odt, 128, 0)))
            launches_per_step += 1 if hp else 0
    traffic, traffic_src = None, None
    if ws == 1 and nnz_total == cfg.nnz and args.out == "f32" and not args.no_hot and R == cfg.rank:
        traffic, traffic_src = traffic_from_profile(args.config)
    for k in [k for k in alto._cache if (k[0] if isinstance(k, tuple) else k) in ("mstream", "hotms")]:
        del alto._cache[k]
    torch.cuda.empty_cache()

    def path_line(name, fn, plan):
        for _ in range(2):
            for n in range(N):
                fn(n)
        _s, pm = time_modes(fn, N, max(3, args.steps // 2), l2, stream)
        ba = [bytes_alg(dims, M, kb, vb, R, fb, n) for n in range(N)]
        return dict(plan, kernel=name, per_mode_ms=pm, nnz_per_s=N * M / (sum(pm) * 1e-3),
                    roofline_frac=sum(ba) / (sum(pm) * 1e-3) / 1e9 / peak)

    paths = {}
    if ws == 1 and not args.skip_paths:
        # the paper's Buffered scheme: K8/K9 slice interval buffers + deterministic pull
        # (the default `auto` API path for large tensors)
        plans["pull"] = plan_leg(build_pull_plans, ("pstream", "pplan", "packed"))
        if mk.mttkrp_pull(alto, fdev, 0, out=outs[0]) is not None:
            paths["buffered_pull"] = path_line("alto::pull_stage_kernel + pull_chunk/seg (alto_pull.cuh), "
                                               "Buffered, deterministic",
                                               lambda n: mk.mttkrp_pull(alto, fdev, n, out=outs[n]), plans["pull"])
            paths["atomic_pull"] = path_line("alto::pull_stage_kernel (alto_pull.cuh), Atomic scheme",
                                             lambda n: mk.mttkrp_pull(alto, fdev, n, out=outs[n], atomic=True),
                                             {})
        for k in [k for k in alto._cache if (k[0] if isinstance(k, tuple) else k) in ("pstream",)]:
            del alto._cache[k]
        torch.cuda.empty_cache()
        # the single mode-agnostic ALTO copy (packed keys + 1-byte sub-tile order per mode)
        if R in (16, 32) and max(lay.bits) <= 31:
            plans["alto_order"] = plan_leg(build_alto_plans, ("packed", "pos"))
            paths["alto_order"] = path_line("alto::planned_kernel (alto_fast.cuh), ALTO order, single copy",
                                            lambda n: mk.mttkrp_stream(alto, fdev, n, out=outs[n], planned="pos"),
                                            plans["alto_order"])
        paths["mode_stream"] = dict(plans["mode_stream"], kernel=kernel_name, per_mode_ms=mode_ms,
                                    nnz_per_s=value, roofline_frac=achieved / peak)
        for k in [k for k in alto._cache if (k[0] if isinstance(k, tuple) else k) in ("pos",)]:
            del alto._cache[k]
        torch.cuda.empty_cache()

    # ---- end to end through the reference-facing API (cli.py:194-203
    # protocol: prepare once; per step host factors in, float64 result out),
    # with the default auto plan (Buffered on every mode -> pull engine) --
    mk.OVERLAP_UPLOADS = True  # pinned inputs are written once, before the timed loop
    parts = at.partition(alto, 16)
    fpin = [torch.from_numpy(f).pin_memory() for f in factors_host]
    opin = [torch.empty((d, R), dtype=torch.float64).pin_memory() for d in dims]
    d2h_stream = torch.cuda.Stream(device=dev)

    def e2e_leg(force):
        pl, fl = [], []
        for n in range(N):
            p = at.plan_conflicts(alto, parts, n, force_strategy=force)
            pl.append(p)
            fl.append(at.apply_boundary_flags(alto, p) if (p.strategy is at.Strategy.ATOMIC
                                                            and p.flag_bit is not None) else alto)

        def e2e_step():
            # every host factor is uploaded once per step (factors_to_device, pinned ->
            # side stream), right before the first mode that reads it, smallest first;
            # the modes then take the device copies (the output mode's own factor is
            # never read: the host tensor stands in for it)
            fd = [None] * N
            for n in range(N):
                for m in sorted((m for m in range(N) if m != n and fd[m] is None), key=lambda m: dims[m]):
                    fd[m] = mk.factors_to_device([fpin[m]])[0]
                o = at.mttkrp_par(fl[n], parts, pl[n], [fd[m] if fd[m] is not None else fpin[m] for m in range(N)],
                                  n, workers=1)
                d2h_stream.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(d2h_stream):
                    opin[n].copy_(o, non_blocking=True)
                o.record_stream(d2h_stream)
            torch.cuda.synchronize()

        for _ in range(2):
            e2e_step()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / args.e2e_steps
        t_e = torch.tensor([t], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        return float(t_e.item()), [p.strategy.value for p in pl]

    e2e_ms, e2e_strat = e2e_leg(None)
    e2e_atomic_ms = None
    if not args.skip_paths:
        e2e_atomic_ms, _ = e2e_leg(at.Strategy.ATOMIC)
    h2d = sum(d * R * fb for d in dims)  # each factor once per step
    d2h = sum(d * R * 8 for d in dims)
    for k in [k for k in alto._cache if (k[0] if isinstance(k, tuple) else k) in ("pstream",)]:
        del alto._cache[k]
    torch.cuda.empty_cache()

    # ---- CP-ALS iteration time (device loop), single GPU only -------------
    cpals = None
    if ws == 1 and not args.skip_cpals:
        from paper_2102_10245_b200.cpd import DeviceCpAls

        cpals = {}
        iters = cfg.als_iters or 10
        rng0 = np.random.default_rng(0)
        t0 = time.perf_counter()
        init = [rng0.random((d, R)) for d in dims]  # cpd_als's initial draw (cpd.py:206-208), host NumPy
        init_ms = (time.perf_counter() - t0) * 1e3
        for backend in ("auto", "atomic"):
            for k in list(alto._cache):
                if (k[0] if isinstance(k, tuple) else k) not in ("packed",):
                    del alto._cache[k]
            torch.cuda.empty_cache()
            torch.cuda.synchronize()
            # cold: plans + initial fit + `iters` sweeps, as cpd_als(tol=0) runs them
            t0 = time.perf_counter()
            st_als = DeviceCpAls(alto, R, seed=0, backend=backend, partitions=16, init_factors=init)
            m0 = st_als.mttkrp(0)
            st_als.fit(m0, 0)
            for _ in range(iters):
                st_als.sweep()
            torch.cuda.synchronize()
            cold = (time.perf_counter() - t0) * 1e3
            # steady state: per-iteration device time (plans built, graphs captured)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            for _ in range(3):
                st_als.sweep()
            c1.record(stream)
            torch.cuda.synchronize()
            cpals[backend] = {"ms_per_iter": c0.elapsed_time(c1) / 3, "iters": iters,
                              f"total_ms_{iters}_iters_incl_plans_and_initial_fit": cold,
                              "host_init_factor_draw_ms": init_ms}
            del st_als
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and ws == 1 and not args.skip_cpu:
        cpu = cpu_baseline_sample(args.config, args.cpu_sample, len(os.sched_getaffinity(0)))

    if rank == 0:
        line = {
            "metric": "MTTKRP nonzeros/sec (mode-averaged)",
            "value": value, "unit": "nnz/s", "n_gpus": ws, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None, "dtype": "f32" if vdt == torch.float32 else "f64",
            "data": f"synthetic (seeded; BASELINE.json {cfg.name} law; generated on {args.gen})",
            "config": {"workload": f"{cfg.name}: {'x'.join(map(str, dims))}, {nnz_total} nnz, {laws_str(cfg)}, "
                                   f"{cfg.values} {cfg.value_dtype} values, rank {R}; step = MTTKRP all {N} modes",
                       "nnz": nnz_total, "rank": R, "key_bits": lay.total_bits, "out_dtype": args.out,
                       "hot_plan": not args.no_hot,
                       "l2": "flushed (256 MB write) before every timed step; keys+values "
                             f"{M * (kb + vb) / 1e6:.0f} MB > 126 MB L2",
                       "parallelism": f"key-range shards x{ws}" if ws > 1 else "1 GPU",
                       "exchange_bytes_per_step": exch_bytes, "shards": shard_info},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_kind,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "bytes_alg_per_launch": tot_b / N, "kernel": kernel_name,
                         "timing": "per-mode CUDA events around the whole MTTKRP call (output zeroing, "
                                   "mode-stream kernel, hot-row reduction)",
                         "per_mode": per_mode,
                         # the access pattern's own ceiling: one factor-row gather per
                         # element and gathered input; tools/gather_probe.cu measures 164-167 G rows/s for
                         # 64-byte rows out of L2 and 40 G rows/s out of HBM (profiles/r02e_gather_probe.txt)
                         "row_gathers_per_s": sum(M * gathers_per_element[n] for n in range(N))
                                              / (sum(mode_ms) * 1e-3),
                         "row_gather_ceiling_per_s": {"l2_resident_64B_rows": 165e9, "hbm_64B_rows": 40e9,
                                                      "source": "profiles/r02e_gather_probe.txt"}},
            "paths": paths,
            "plans": plans,
            "e2e": {"value": N * nnz_total / (e2e_ms * 1e-3), "unit": "nnz/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "plan": e2e_strat,
                    "api": "paper_2102_10245_b200.mttkrp_par with the default (auto) conflict plan over 16 "
                           "partitions (Buffered on every mode -> K8/K9 pull engine); per step every pinned host "
                           "float32 factor is uploaded once (factors_to_device) and every mode's float64 result "
                           "is copied to pinned host memory on a copy stream; PCIe-bound (55 GB/s per direction)",
                    "atomic_plan_value": (N * nnz_total / (e2e_atomic_ms * 1e-3)) if e2e_atomic_ms else None},
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clk.summary(),
            "build_ms": build_ms, "gen_s": t_gen,
            "cpals": cpals,
            "cpals_ms_per_iter": cpals["auto"]["ms_per_iter"] if cpals else None,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--rank", type=int, default=0, help="override the config's rank (rank sweep)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--skip-paths", action="store_true", help="only the headline mode-stream step")
    ap.add_argument("--nnz", type=int, default=0, help="override nnz (testing)")
    ap.add_argument("--tile", type=int, default=1024)
    ap.add_argument("--cpu-sample", type=int, default=2_000_000)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-cpals", action="store_true")
    ap.add_argument("--no-hot", action="store_true", help="disable the hot-row plan (A/B)")
    ap.add_argument("--l2-hot-mb", type=float, default=None,
                    help="L2 residency budget (MB) for the gathered factors (mttkrp.MS_L2_HOT_MB; A/B)")
    ap.add_argument("--out", default=None, choices=["f32", "f64"],
                    help="MTTKRP output dtype of the bench step (default: the config's value dtype)")
    ap.add_argument("--gen", default="device", choices=["device", "host"],
                    help="synthetic input generator: torch on the GPU (fast) or the NumPy stream of the parity tests")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
