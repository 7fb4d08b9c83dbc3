#!/usr/bin/env python
"""bench.py — RT-DetMCD fit + flag throughput on B200 (BASELINE.json `metric`).

One step = one whole pass of the hot path over
one batch of synthetic input: standardise, starts, refinement, C-steps,
raw fit (+ aggregation for q > 1), reweighting and the flag pass over all n
rows.  Default workload: BASELINE config 4 (n = 8,000,000, p = 40, h = 0.75 n,
q = 8 contiguous per-shard blocks) on one GPU; inputs (2.56 GB) are larger
than L2 (126 MB), so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

Prints ONE JSON line (rank 0).  `value` = observations/s over all ranks with X
resident in HBM; `e2e` = the same through the C ABI with pinned HOST buffers
(H2D of X and D2H of the flags inside the timed region); `roofline` = the
C-step distance pass (the north-star kernel) measured live with CUDA events
on the library stream; `cpu_baseline` = the CPU oracle on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_NAMES = {1: "cfg1_n1000_p5", 2: "cfg2_n100k_p10", 3: "cfg3_n1M_p20", 4: "cfg4_n8M_p40_q8", 5: "cfg5_n20k_p8"}
METRIC = "observations/sec fitted+flagged (RT-DetMCD, fp64)"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def make_workload(cfg: int, n: int | None = None):
    from paper_1910_05615_b200 import datagen
    d = datagen.make_config(cfg, n=n)
    return d


SAMPLE_N = {1: 1000, 2: 100_000, 3: 100_000, 4: 100_000, 5: 20_000}  # one sample size for both CPU legs


def cpu_baseline(cfg: int, sample_n: int | None = None):
    """The oracle, as it stands, on a bounded sample of the same workload (rank 0, N = 1 only).
    `cores` = the cores the run actually kept busy (process CPU time / wall time: numpy's BLAS threads in
    the matrix products, one core elsewhere); `blas_threads` = the BLAS pool size."""
    from threadpoolctl import threadpool_info

    from oracle import fit as ofit
    from paper_1910_05615_b200 import datagen
    if sample_n is None:
        sample_n = SAMPLE_N[cfg]
    d = datagen.make_config(cfg, n=sample_n)
    q = d.q if cfg == 4 else 1
    h = int(math.floor(0.75 * sample_n)) if cfg == 4 else d.h
    c0, t0 = time.process_time(), time.perf_counter()
    ofit.fit(d.X, h=h, q=q, seed=191005615, log_transform=d.log_transform,
             partition_mode="contiguous" if cfg == 4 else "permute")
    dt = time.perf_counter() - t0
    cpu = time.process_time() - c0
    threads = max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    return {"value": sample_n / dt, "unit": "obs/s", "cores": round(cpu / dt, 2), "blas_threads": int(threads),
            "kind": "oracle",
            "sample": f"config {cfg} recipe at n={sample_n} (q={q}), one fit+flag, {dt:.1f} s wall, {cpu:.1f} s CPU"}


def run_reference(args, rank: int, world: int):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only)."""
    if rank != 0:
        return
    cfg = args.config
    times = []
    sample_n = args.ref_sample or SAMPLE_N[cfg]
    for s in range(args.warmup + args.steps):
        cb = cpu_baseline(cfg, sample_n)
        if s >= args.warmup:
            times.append(sample_n / cb["value"])
    ms = 1e3 * float(np.mean(times))
    value = sample_n / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": "obs/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": CONFIG_NAMES[cfg], "sample_rows": sample_n},
            "cpu_baseline": {"value": value, "unit": "obs/s", "cores": cb["cores"], "blas_threads": cb["blas_threads"],
                             "kind": "oracle", "sample": cb["sample"]},
            "e2e": {"value": value, "unit": "obs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_stream(args, local: int):
    """Config 5: the real-time stream (BASELINE.json configs[4]) -- B consecutive batches of
    20,000 x 8 (ln of lognormal), each one fit + flag; per-batch latency p50 / p99.

    X of every batch is resident in HBM before the timed region; each batch is timed with
    CUDA events on the launching stream (device) and with the host clock around the
    synchronous call (wall).  `e2e` repeats the stream from pinned host batches (H2D of X
    and D2H of the flags inside each call)."""
    import torch

    from paper_1910_05615_b200 import api, datagen
    nb = args.steps
    t0 = time.perf_counter()
    batches = [datagen.make_config(5, batch=b) for b in range(nb)]
    gen_s = time.perf_counter() - t0
    n, p = batches[0].X.shape
    h = batches[0].h
    Xd = [torch.from_numpy(b.X).to(f"cuda:{local}") for b in batches]
    stream = torch.cuda.current_stream()

    flags_d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local}")

    def one(X, **kw):
        kw.setdefault("out_buffers", {"flags": flags_d})
        return api.fit(X, h=h, q=1, log_transform=True, outputs=(), **kw)

    for b in range(args.warmup):
        one(Xd[b % nb])
    torch.cuda.synchronize()
    k0, s0 = api.counters()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nb)]
    wall = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for b in range(nb):
            w0 = time.perf_counter()
            evs[b][0].record(stream)
            res = one(Xd[b])
            evs[b][1].record(stream)
            wall.append(1e3 * (time.perf_counter() - w0))
        g1.record(stream)
        torch.cuda.synchronize()
    k1, s1 = api.counters()
    # warm-started stream: batch b's C-steps start from batch b-1's reweighted fit
    # (the previous batch's own result from the chain; batch 0's cold fit seeds it)
    wdev = []
    prev = (res0 := one(Xd[0])).mu_rew, res0.sigma_rew
    torch.cuda.synchronize()
    for b in range(1, nb):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rw = one(Xd[b], warm_start=prev)
        e1.record(stream)
        e1.synchronize()
        wdev.append(e0.elapsed_time(e1))
        prev = (rw.mu_rew, rw.sigma_rew)
    # kernel breakdown / roofline from a separate profiled pass (per-kernel events stay out of the latencies)
    nprof = min(nb, 100)
    api.set_profiling(True, device=local)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for b in range(nprof):
        one(Xd[b])
    pe1.record(stream)
    torch.cuda.synchronize()
    prof = api.profile(device=local)
    api.set_profiling(False, device=local)
    prof_ms = pe0.elapsed_time(pe1)
    dev_ms = np.array([a.elapsed_time(b) for a, b in evs])
    total_ms = g0.elapsed_time(g1)
    value = n * nb / (total_ms / 1e3)
    # e2e: pinned host batch in, host flags out, through the same public call
    e2e = None
    if not args.no_e2e:
        Xh = [torch.from_numpy(b.X).pin_memory() for b in batches]
        fl = torch.empty(n, dtype=torch.uint8).pin_memory()
        one(Xh[0], out_buffers={"flags": fl})
        torch.cuda.synchronize()
        e_wall = []
        w_start = time.perf_counter()
        for b in range(nb):
            w0 = time.perf_counter()
            one(Xh[b], out_buffers={"flags": fl})
            e_wall.append(1e3 * (time.perf_counter() - w0))
        e_tot = time.perf_counter() - w_start
        e2e = {"value": n * nb / e_tot, "unit": "obs/s", "h2d_bytes_per_step": int(n * p * 8),
               "d2h_bytes_per_step": int(n),
               "latency_ms": {"p50": float(np.percentile(e_wall, 50)), "p99": float(np.percentile(e_wall, 99))}}
    roof = _roofline(prof, prof_ms, 5)
    cb = None if args.no_cpu_baseline else cpu_baseline(5)
    line = {"metric": METRIC, "value": value, "unit": "obs/s", "n_gpus": 1, "steps": nb, "warmup": args.warmup,
            "ms_per_step": total_ms / nb, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[5], "n": int(n), "p": int(p), "h": int(h), "q": 1, "batches": nb,
                       "log_transform": True, "l2": "batch (1.28 MB) is L2-resident: latency-bound by design",
                       "batch_gen_s": gen_s, "parallelism": "replicas only (batches are independent)"},
            "latency_ms": {"p50": float(np.percentile(dev_ms, 50)), "p99": float(np.percentile(dev_ms, 99)),
                           "wall_p50": float(np.percentile(wall, 50)), "wall_p99": float(np.percentile(wall, 99)),
                           "max": float(dev_ms.max())},
            "warm_start": {"latency_ms": {"p50": float(np.percentile(wdev, 50)), "p99": float(np.percentile(wdev, 99))},
                           "value": n * len(wdev) / (sum(wdev) / 1e3), "unit": "obs/s",
                           "note": "each batch's C-steps start from the previous batch's reweighted fit "
                                   "(PAPER.md:1038-1043); initial estimators and refinement skipped"}
            if wdev else None,
            "e2e": e2e, "roofline": roof, "cpu_baseline": cb, "gpu_launches": int(k1 - k0), "cub_sorts": int(s1 - s0),
            "clocks": clk.summary(), "breakdown": _breakdown(prof, nprof),
            "fit": {"start_steps": [int(x) for x in res.start_steps]}}
    return line


def quick_fit(cfg: int, local: int, steps: int, warmup: int):
    """A sub-record of the default bench line: config `cfg` fitted + flagged on this GPU (X resident),
    CUDA events over `steps` fits after `warmup`, plus the distance-pass roofline from a profiled pass."""
    import torch

    from paper_1910_05615_b200 import api
    d = make_workload(cfg)
    n, p = d.X.shape
    Xd = torch.from_numpy(d.X).to(f"cuda:{local}")
    fl = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local}")

    def step():
        return api.fit(Xd, h=d.h, q=d.q, log_transform=d.log_transform, outputs=(), out_buffers={"flags": fl})
    for _ in range(warmup):
        step()
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    api.set_profiling(True, device=local)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    prof = api.profile(device=local)
    api.set_profiling(False, device=local)
    del Xd
    return {"workload": CONFIG_NAMES[cfg], "n": int(n), "p": int(p), "h": int(d.h), "q": int(d.q),
            "value": n * steps / (ms / 1e3), "unit": "obs/s", "ms_per_step": ms / steps, "steps": steps,
            "warmup": warmup, "roofline": _roofline(prof, p0.elapsed_time(p1), cfg),
            "breakdown": {k: v for k, v in list(_breakdown(prof, steps).items())[:6]}}


def _fp64_peak():
    """FP64 tensor-pipe (DMMA m8n8k4) peak: profiles/fp64_peak.json written by tools/fp64_peak on a B200
    (MEASURED_PEAKS.json has no fp64 entry), else the value DESIGN.md records from that tool."""
    try:
        j = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        return float(j["dmma_tflops"]), "measured (profiles/fp64_peak.json, tools/fp64_peak.cu DMMA burst)"
    except Exception:
        return 37.0, "measured earlier with tools/fp64_peak.cu (DMMA burst at 1965 MHz, DESIGN.md section 6)"


def _traffic(cfg: int):
    """ncu DRAM bytes per algorithmic byte of the distance pass (profiles/r02_dist_traffic.json, from one
    `ncu --set full` capture of the same kernel on the same workload)."""
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "r02_dist_traffic.json")))
        e = tj.get(CONFIG_NAMES[cfg])
        return (e["dram_bytes"] / e["algorithmic_bytes"], tj.get("source")) if e else (None, None)
    except Exception:
        return None, None


def _roofline(prof: dict, ms_local: float, cfg: int):
    """The C-step distance pass (north-star kernel, k_dist_tma): per launch, its ALGORITHMIC bytes (every
    block an item reads once -- the two starts of a block share the tile -- plus one d^2 per row and
    start) and flops (p(p+1) + 2p per row and start) over the average launch time from CUDA events on the
    library stream, against the measured HBM copy peak and the measured FP64 tensor (DMMA) peak.
    `bound` is the resource at the higher fraction; both are reported."""
    peaks = _peaks()
    hbm_peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if hbm_peak else "fallback (B200_PROFILING.md 6650 GB/s)"
    hbm_peak = hbm_peak or 6650.0
    if "dist" not in prof or prof["dist"]["ms"] <= 0:
        return None
    dstat = prof["dist"]
    sec = dstat["ms"] / 1e3
    gbs = dstat["bytes"] / sec / 1e9
    tfs = dstat.get("flops", 0.0) / sec / 1e12
    fpk, fsrc = _fp64_peak()
    hbm = {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak, "peak_source": peak_src}
    ten = {"achieved": tfs, "peak": fpk, "unit": "TFLOP/s", "frac": tfs / fpk, "peak_source": fsrc,
           "pipe": "FP64 tensor (DMMA m8n8k4)"}
    main = ten if ten["frac"] > hbm["frac"] else hbm
    L = dstat["launches"]
    out = {"bound": "tensor" if main is ten else "hbm", "achieved": main["achieved"], "peak": main["peak"],
           "unit": main["unit"], "frac": main["frac"], "traffic": None,
           "kernel": "k_dist_tma (C-step distance pass, TMA-fed, two starts per tile)",
           "peak_source": main["peak_source"], "hbm": hbm, "fp64_tensor": ten,
           "launches": L, "avg_launch_ms": dstat["ms"] / L, "bytes_per_launch": dstat["bytes"] / L,
           "flops_per_launch": dstat.get("flops", 0.0) / L,
           "per_start_definition": {"GBps": dstat.get("eff_bytes", 0.0) / sec / 1e9,
                                    "frac": dstat.get("eff_bytes", 0.0) / sec / 1e9 / hbm_peak,
                                    "note": "SURVEY 8(d): (8p + 8) bytes per row per start, as if every start "
                                            "streamed its block alone"},
           "ms_share_of_step": dstat["ms"] / ms_local}
    ratio, src = _traffic(cfg)
    if ratio is not None:
        out["traffic"] = ratio * out["bytes_per_launch"]
        out["traffic_source"] = src
    return out


def _breakdown(prof: dict, steps: int):
    return {k: {"ms_per_step": v["ms"] / steps, "launches_per_step": v["launches"] / steps,
                "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 and v["bytes"] > 0 else None}
            for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}


def _relaunch(n: int):
    """`python bench.py --gpus N` without torchrun: start N ranks on this node (127.0.0.1 rendezvous)."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} needs {n} GPUs, this node has {have}"}), flush=True)
        sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default 20; config 5: 1000 batches)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--n", type=int, default=0, help="override rows (debug only; not a bench line)")
    ap.add_argument("--no-sub", action="store_true", help="skip the config-3 / config-5 sub-records")
    ap.add_argument("--stream-batches", type=int, default=1000, help="batches of the config-5 sub-record")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.steps is None:
        args.steps = 1000 if args.config == 5 else 20  # >= 0.6 s timed at config 4: several clock samples

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        _relaunch(args.gpus)          # one process per GPU: re-exec under torchrun (never a silent 1-rank run)
        return
    if args.impl != "reference" and world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_1910_05615_b200 import api

    cfg = args.config
    if cfg == 5:
        if rank == 0:
            print(json.dumps(run_stream(args, local)), flush=True)  # replicas only (independent batches)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return
    d = make_workload(cfg, n=args.n or None)
    n, p = d.X.shape
    q = d.q
    h = d.h
    # config 4: rows sharded over the GPUs with per-shard DetMCD (BASELINE.json configs[3]) ->
    # contiguous blocks at every GPU count, so N = 1, 2, 4, 8 compute the same estimate
    part = 1 if cfg == 4 else 0
    if world > 1:
        # rtdetmcd_fit_sharded over NCCL: the library exchanges columns, block records and reweighting sums
        from paper_1910_05615_b200 import distributed as rtd_dist
        runner = rtd_dist.ShardedFit(d.X, h=h, q=q, log_transform=d.log_transform, rank=rank, world=world,
                                     device=local)
        step = runner.step
        n_rows_total = n
    else:
        Xd = torch.from_numpy(d.X).to(f"cuda:{local}")

        flags_d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local}")

        def step():  # the caller's device buffer receives the flags (no allocation inside the timed steps)
            return api.fit(Xd, h=h, q=q, seed=191005615, log_transform=d.log_transform, partition=part,
                           outputs=(), out_buffers={"flags": flags_d})
        n_rows_total = n

    # warm-up (also sizes the workspace)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    prof_ctx = runner.ctx if world > 1 else None
    k0, s0 = api.counters()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    stream = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            res = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    k1, s1 = api.counters()
    ms_local = ev0.elapsed_time(ev1)
    # per-kernel-class device times from a separate profiled pass (its events stay out of the timed steps)
    api.set_profiling(True, device=local, ctx=prof_ctx)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for _ in range(args.steps):
        step()
    pe1.record(stream)
    torch.cuda.synchronize()
    prof = api.profile(device=local, ctx=prof_ctx)
    api.set_profiling(False, device=local, ctx=prof_ctx)
    prof_ms = pe0.elapsed_time(pe1)
    ms = ms_local
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_local], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = n_rows_total * args.steps / (ms / 1e3)

    # e2e: the same step through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e and world > 1:
        # every rank: its pinned host rows in, its flags out, through rtdetmcd_fit_sharded (the library copies
        # the rows to the device inside the call); time = max over ranks of the device-side span
        import torch.distributed as dist
        a, b, _, _ = rtd_dist.shard_rows(n, q, world, rank)
        Xh = torch.from_numpy(np.ascontiguousarray(d.X[a:b])).pin_memory()
        fl = torch.empty(b - a, dtype=torch.uint8).pin_memory()

        def hstep():
            return api.fit_sharded(Xh, n, runner.ctx, h=h, q=q, log_transform=d.log_transform, outputs=(),
                                   out_buffers={"flags": fl})
        hstep()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            hstep()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        t = torch.tensor([wall], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
        e2e = {"value": n * args.steps / wall, "unit": "obs/s", "h2d_bytes_per_step": int(n * p * 8),
               "d2h_bytes_per_step": int(n),
               "api": "rtdetmcd_fit_sharded per rank from pinned host rows (H2D + D2H of flags inside each call), "
                      "max over ranks"}
    if not args.no_e2e and world == 1:
        # K host batches through rtdetmcd_fit_batches: every step copies its batch from pinned host memory
        # and reads its flags back; batch k+1's copy runs on the library's copy stream during batch k's fit
        Xh = torch.from_numpy(d.X).pin_memory()
        fl = torch.empty(n, dtype=torch.uint8).pin_memory()
        kw = dict(h=h, q=q, seed=191005615, log_transform=d.log_transform, partition=part, outputs=(),
                  out_buffers={"flags": fl})
        api.fit_batches([Xh, Xh], **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        api.fit_batches([Xh] * args.steps, **kw)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ems = max(e0.elapsed_time(e1), wall * 1e3)
        e2e = {"value": n * args.steps / (ems / 1e3), "unit": "obs/s", "h2d_bytes_per_step": int(n * p * 8),
               "d2h_bytes_per_step": int(n),
               "api": "rtdetmcd_fit_batches over K pinned host batches (H2D of batch k+1 overlaps the fit of batch k)"}

    roof = _roofline(prof, prof_ms, cfg)
    breakdown = _breakdown(prof, args.steps)

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(cfg)

    # sub-records (N = 1): config 3, the HBM-scale p = 20 case, and config 5, the real-time stream
    # (BASELINE.json configs[2], configs[4]); parity-test workloads, reported beside the headline
    sub = None
    if rank == 0 and world == 1 and not args.no_sub and cfg == 4:
        import copy
        sub = {"cfg3": quick_fit(3, local, 10, 3)}
        sa = copy.copy(args)
        sa.steps, sa.warmup, sa.no_cpu_baseline, sa.no_e2e = args.stream_batches, 3, True, False
        sl = run_stream(sa, local)
        sub["cfg5_stream"] = {k: sl[k] for k in ("value", "unit", "ms_per_step", "latency_ms", "warm_start", "e2e",
                                                 "gpu_launches", "cub_sorts", "roofline")}
        sub["cfg5_stream"]["batches"] = sa.steps

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "obs/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": CONFIG_NAMES[cfg], "n": int(n), "p": int(p), "h": int(h), "q": int(q),
                           "partition": "contiguous per-shard blocks" if part else "feistel",
                           "l2": "inputs larger than L2 (no flush)",
                           "parallelism": f"rows over {world} GPU(s)" + (
                               " (rtdetmcd_fit_sharded, NCCL inside the library)" if world > 1 else "")},
                "e2e": e2e, "roofline": roof, "cpu_baseline": cb,
                "gpu_launches": int((k1 - k0)), "cub_sorts": int(s1 - s0),
                "clocks": clk.summary(), "breakdown": breakdown,
                "fit": {"block_chosen": [int(x) for x in res.block_chosen] if hasattr(res, "block_chosen") else None,
                        "start_steps": [int(x) for x in res.start_steps] if hasattr(res, "start_steps") else None},
                "sub": sub}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
