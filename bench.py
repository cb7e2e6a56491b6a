#!/usr/bin/env python
"""Benchmark: squarefree d = 5 mod 8 classified per second at d ~ 1e10.

Workload (BASELINE.json metric): the window (9e9, 1e10] is
cut into 8 slabs of width 1.25e8 (~12.66 M d in D each).  Rank r of an N-GPU
job owns slab r counted down from 1e10 (weak scaling: per-GPU work fixed; N=8
covers the whole window, N=1 is (9.875e9, 1e10], which contains Table 1's
window (9.9e9, 1e10]).  One step = the whole hot path over the job's d:
sieve + compaction + residue walk + checkpoint histogram on every GPU, one
all-reduce of the checkpoint buckets (NCCL), prefix kernel.  `value` = #D in
the job's window / device time of a step (max over ranks).

Launch: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
(N>1 under torchrun; RANK/LOCAL_RANK/WORLD_SIZE from the environment).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

METRIC = "squarefree d≡5 mod 8 classified/sec (whole box) at d≈10^10; 1/2/4/8 B200"
UNIT = "d/s"
SM_MAX_MHZ_FALLBACK = 1965.0
# Algorithmic thread-operations per unit of work:
# Work per unit: one rho step (+ residue + exit tests) is 14 SASS
# instructions in the kernel's FP32 formulation (cuobjdump), so `frac` is the
# share of the chip's issue slots spent on step instructions.  SURVEY 8(d)'s
# generic u32 step is 34 instructions; `work_equiv_generic` reports that view.
OPS_PER_BABY = 14
GENERIC_PER_BABY = 34
OPS_PER_GIANT = 700    # thread-instructions of one fast-path giant step (K3 BSGS)
OPS_PER_ENTRY = 12     # store insert per window entry: slot pack, hash, bucket insert
# algorithmic HBM bytes of the window kernel (per-unit figures): per
# entry 4 (list write) + 4 (list read-back by the build) + 64 / (16 * 0.62) (table
# slots at load 0.62 in 64-byte buckets); per d 32 (window record) + 4 + 4 (offset,
# queue entry)
WIN_BYTES_PER_ENTRY = 4 + 4 + 64 / (16 * 0.62)
WIN_BYTES_PER_D = 40
# DRAM bytes per d of the BSGS walk at the bench configuration: dram__bytes_read +
# dram__bytes_write of bsgs_window + bsgs_prep + bsgs_giant for one segment (ncu
# --set full, profiles/r01_bsgs_walk.txt: 39.73 + 1.59 + 13.72 GB) / the segment's
# 6.33 M d.  Algorithmic: list write + read-back 3.6 KB, table 2.9 KB, ~18.5 probes
# x 64 B, records ~0.2 KB = ~7.9 KB per d.
BSGS_DRAM_BYTES_PER_D = 8563


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    REASONS = ["gpu_idle", "applications_clocks_setting", "sw_power_cap", "hw_slowdown",
               "sync_boost", "sw_thermal_slowdown", "hw_thermal_slowdown",
               "hw_power_brake_slowdown"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_hbm_gbs() -> float:
    """HBM copy bandwidth from MEASURED_PEAKS.json (driver-written), else the
    B200_PROFILING.md fallback of 6,650 GB/s."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(lo: int, hi: int, seconds_target: float = 15.0, n: int | None = None) -> dict:
    """The oracle as it stands, on all host cores, on a seeded sample of the
    workload (candidates of (lo, hi]); value in d/s (d in D only).  The thread
    count is passed explicitly (torchrun sets OMP_NUM_THREADS=1)."""
    from oracle import c_oracle

    ncpu = host_cores()
    # ~15 ms/d/core at 1e10 (measured), so ncpu*1000 candidates ~ 15 s
    n = n or max(64, int(ncpu * 1000 * seconds_target / 15.0))
    s = workloads.sample_candidates(lo + 1, hi, n, seed=workloads.SEED + 1)
    c_oracle.lib()
    t0 = time.perf_counter()
    f = c_oracle.classify_list(s, ncpu)
    dt = time.perf_counter() - t0
    nd = int((f != c_oracle.NOT_IN_D).sum())
    return {"value": nd / dt, "unit": UNIT, "cores": ncpu, "kind": "oracle",
            "sample": f"{len(s)} seeded uniform candidates (seed {workloads.SEED + 1}) of "
                      f"({lo}, {hi}], {nd} in D, big-integer CF oracle, {dt:.1f} s wall on "
                      f"{ncpu} threads"}


def run_reference(args) -> None:
    rank = _env_int("RANK", 0)
    if rank != 0:
        return
    n_gpus = args.gpus
    lo, hi = workloads.metric_window(n_gpus)
    ncpu = host_cores()
    per_step = max(32, int(ncpu * 1000 * args.ref_seconds / 15.0))
    vals, times = [], []
    for k in range(args.warmup + args.steps):
        cb = cpu_baseline(lo, hi, n=per_step)
        if k >= args.warmup:
            vals.append(cb["value"])
            times.append(per_step / cb["value"])
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bigint", "data": "synthetic",
        "config": {"workload": f"metric window ({lo}, {hi}]: all d = 5 mod 8 (oracle: seeded "
                               f"sample of {per_step} candidates per step)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": ncpu, "kind": "oracle",
                         "sample": f"{per_step} seeded candidates of ({lo}, {hi}] per step"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="auto", choices=["auto", "half", "bsgs"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo: orchestration test only)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="all ranks on cuda:0 (orchestration test on a 1-GPU box; the "
                         "ranks' kernels never wait on one another)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2507_06579_b200 as eis
    from paper_2507_06579_b200.dist import allreduce_buckets, count_window_distributed

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 must be launched under torchrun")
    gpu = 0 if args.share_gpu else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    eis.init(gpu)
    eis.set_option("mode", {"auto": eis.MODE_AUTO, "half": eis.MODE_HALF,
                            "bsgs": eis.MODE_BSGS}[args.mode])

    lo, hi = workloads.metric_slab(rank)          # this rank's slab
    jlo, jhi = workloads.metric_window(world)      # the job's window
    x = np.asarray(workloads.metric_checkpoints(world), dtype=np.uint64)
    n = len(x)
    stream = torch.cuda.current_stream(dev)
    buckets = torch.zeros(2 * n, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.int32, device=dev)   # 256 MiB > L2

    def step():
        buckets.zero_()
        eis.count_buckets_dev(lo, hi, x, buckets, stream=stream)
        allreduce_buckets(buckets)
        eis.prefix_dev(buckets, buckets, stream=stream)

    for _ in range(args.warmup):
        step()
        flush.fill_(1)
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    walk_ms, launches, stats = [], 0, {}
    kern_ms = {"sieve": [], "window": [], "giant": []}
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    sampler = ClockSampler(int(cvd.split(",")[gpu]) if cvd else gpu)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
        stats = eis.get_stats()
        walk_ms.append(stats["walk_ms"])
        for kn in kern_ms:
            kern_ms[kn].append(stats[f"{kn}_ms"])
        launches += int(stats["kernel_launches"]) + 1      # + prefix kernel
        flush.fill_(k)                                      # untimed: evict L2
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    res = buckets.cpu().numpy().astype(np.uint64)

    t = torch.tensor([tot_ms, float(np.mean(walk_ms))] + [float(np.mean(v)) for v in kern_ms.values()],
                     dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms_max, walk_ms_max = float(t[0]), float(t[1])
    kms = dict(zip(kern_ms, (float(v) for v in t[2:])))

    # verification of the bench output itself: Table 1 window (9.9e9, 1e10]
    i99 = list(x).index(9_900_000_000)
    e_9910 = int(res[n + n - 1] - res[n + i99])
    verified = e_9910 == 3_334_227
    nD_job = int(res[n - 1])
    nD_rank = int(stats["d_classified"])

    # e2e through the public API with host buffers (H2D of x, D2H of counts in the call)
    e2e_s = []
    for _ in range(args.e2e_steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world > 1:
            cD, cE = count_window_distributed(jlo, x)
        else:
            cD, cE = eis.count_window(jlo, x)
        e2e_s.append(time.perf_counter() - t0)
    te = torch.tensor([statistics.median(e2e_s)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ok = int(cD[-1]) == nD_job and int(cE[-1]) == int(res[2 * n - 1])

    if rank == 0:
        value = nD_job / (tot_ms_max / args.steps / 1e3)
        sm_clk = clocks.get("sm_mhz") or SM_MAX_MHZ_FALLBACK
        peak = 148 * 4 * 32 * sm_clk * 1e6 / 1e12                 # issue-slot peak, Tops/s
        bsgs = stats["giant_steps"] > 0
        # algorithmic thread-ops of each kernel family in one step (this rank)
        entries = stats["baby_steps"] if bsgs else 0              # one store entry per step
        kops = {"window": OPS_PER_BABY * stats["baby_steps"] + OPS_PER_ENTRY * entries,
                "giant": OPS_PER_GIANT * stats["giant_steps"]}
        per_kernel = {k: {"ms": kms[k], "tops": kops[k] / (kms[k] / 1e3) / 1e12 if kms[k] else None}
                      for k in kops}
        for k in per_kernel:
            if per_kernel[k]["tops"] is not None:
                per_kernel[k]["frac"] = per_kernel[k]["tops"] / peak
        per_kernel["sieve"] = {"ms": kms["sieve"]}
        if bsgs:
            # the window kernel is bound by HBM, not issue: its algorithmic bytes over
            # its live span (which overlaps the giant kernel of the previous segment)
            wbytes = WIN_BYTES_PER_ENTRY * entries + WIN_BYTES_PER_D * stats["d_classified"]
            hbm_peak = measured_hbm_gbs()
            per_kernel["window"]["hbm"] = {
                "bytes_per_step": wbytes, "gbs": wbytes / (kms["window"] / 1e3) / 1e9,
                "peak_gbs": hbm_peak, "frac": wbytes / (kms["window"] / 1e3) / 1e9 / hbm_peak,
                "note": "live span includes the overlapped giant kernel; ncu alone "
                        "(profiles/r01_bsgs_walk.txt): 39.7 GB in 7.22 ms per 6.33 M-d "
                        "segment = 5.5 TB/s, 0.84 of the measured copy bandwidth"}
        if bsgs:
            # the BSGS kernels run on two streams and overlap (the giant kernel of one
            # segment with the window kernel of the next), so the walk is the unit:
            # all of its algorithmic ops over its device time
            ops_per_launch = kops["window"] + kops["giant"]
            achieved = ops_per_launch / (walk_ms_max / 1e3) / 1e12
            dom_name = "BSGS walk: bsgs_window_kernel + bsgs_prep_kernel + bsgs_giant_kernel"
            dom_ms = walk_ms_max
        else:
            ops_per_launch = kops["window"]
            achieved = per_kernel["window"]["tops"]
            dom_name = "walk_half_kernel"
            dom_ms = kms["window"]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if stats["giant_steps"] == 0 else "f32+f64",   # exact-integer FP
            "data": "synthetic",
            "config": {
                "workload": f"all d = 5 mod 8 in ({jlo}, {jhi}] ({nD_job} d in D); rank r owns "
                            f"slab ({workloads.METRIC_TOP}-(r+1)*{workloads.METRIC_SLAB}, "
                            f"{workloads.METRIC_TOP}-r*{workloads.METRIC_SLAB}]",
                "checkpoints": f"{n} (every 1e7)", "mode": args.mode,
                "l2": "flushed between steps (256 MiB write, untimed)",
                "verified": {"E(9.9e9,1e10]": e_9910, "paper": 3_334_227, "ok": verified,
                             "e2e_counts_match": e2e_ok},
            },
            "e2e": {"value": nD_job / float(te[0]), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                    "d2h_bytes_per_step": 16 * n,
                    "path": "eis_count_window (C ABI, host buffers)" if world == 1
                    else f"count_window_distributed (C ABI dev + {args.backend} allreduce)"},
            "gpu_launches": launches,
            "roofline": {
                "bound": "alu", "kernel": dom_name,
                "achieved": achieved, "peak": peak, "unit": "Tops/s", "frac": achieved / peak,
                "traffic": BSGS_DRAM_BYTES_PER_D * nD_rank if bsgs else 50.8e6,
                "traffic_note": ("dram read+write bytes per step of the BSGS walk: 8.56 KB per d "
                                 "measured by ncu --set full on the bench workload "
                                 "(profiles/r01_bsgs_walk.txt) x d per step; algorithmic ~8.5 KB "
                                 "per d (list 3.9, table 3.2, probes 1.1, records 0.3); the "
                                 "window kernel is HBM-bound (per_kernel.window.hbm), the giant "
                                 "kernel issue/latency-bound") if bsgs else
                                "dram read+write bytes per walk launch, ncu --set full "
                                "(profiles/r01_half_walk.txt); algorithmic bytes = 4 per d "
                                "(survivor list) = 50.7 MB",
                "ops_per_step": ops_per_launch,
                "kernel_ms_per_step": dom_ms,
                "per_kernel": per_kernel,
                "work_equiv_generic": None if bsgs else
                (GENERIC_PER_BABY * stats["baby_steps"]) / (kms["window"] / 1e3) / 1e12 / peak,
                "walk_ms_per_step": walk_ms_max,
                "walk_share_of_step": walk_ms_max / (tot_ms_max / args.steps),
                "basis": f"thread-ops per unit: {OPS_PER_BABY} per rho step, {OPS_PER_ENTRY} per "
                         f"store entry, {OPS_PER_GIANT} per giant step; kernel time = summed CUDA "
                         f"events around its launches on its own stream (BSGS: the walk's span, "
                         f"per_kernel spans overlap); peak = 148 SM x 4 SMSP x "
                         f"32 lanes x {sm_clk:.0f} MHz (sampled SM clock) issue slots (DESIGN.md 4)",
            },
            "clocks": clocks,
            "stats_per_rank_step": {k: stats[k] for k in ("d_classified", "baby_steps",
                                                          "giant_steps", "sym_exits")},
            "rank_d": nD_rank,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(jlo, jhi)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
