#!/usr/bin/env python3
"""bench.py -- batched 1D C2C FFT on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fftc|reference] [--workload c2|c1|c3|c4]

Workload (default, BASELINE.json configs[1]): the power-of-two sweep
N = 2^3 ... 2^12, batch = 2^26/N (2^26 complex64 = 512 MiB per buffer, larger
than the 126 MB L2, so no flush is needed; smaller workloads such as C1 get an L2 flush
between timed steps), values U[-1,1) from seed 0, forward
AND inverse.  One step = the whole sweep = 20 fftc_execute calls (10 sizes x 2
signs), each a full pass of the hot path (stage-in, Stockham stages, stage-out).

value  = sum over the step of 5 N log2(N) batch flops / device time (GFLOP/s),
         whole job (all ranks) / max over ranks.
e2e    = the same metric through fftc_execute_host: pinned host input ->
         device -> transform -> host output, copies inside the timed region.
roofline: the fused Stockham kernel family (every launch of the step is one);
         achieved = algorithmic bytes per launch (16 B per complex element:
         8 read + 8 written) / mean launch time (CUDA events on
         the launch stream); peak = MEASURED_PEAKS.json hbm_gbs.
cpu_baseline: the oracle's recursive Cooley-Tukey (oracle/, fp64, OpenMP) on a
         bounded sample of the same workload (rank 0, N=1 only).

Multi-GPU (torchrun): every rank runs the full sweep on its own seeded batch
(weak scaling: transforms are independent, no data-path collective); barrier +
synchronize around the timed region, max over ranks via all_reduce(MAX).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched 1D C2C FFT GFLOP/s (5N·log2N) and HBM GB/s vs peak, 1/2/4/8 B200"
UNIT = "GFLOP/s"
ELEMS = 1 << 26


def workloads(name):
    """-> (description, [(N, batch, sign, dist)])"""
    if name == "c2":
        jobs = [(1 << k, ELEMS >> k, s, "uniform") for k in range(3, 13) for s in (-1, 1)]
        return ("C2 pow2 sweep N=2^3..2^12, batch=2^26/N, fwd+inv", jobs)
    if name == "c1":
        return ("C1 N=64 batch=4096 fwd", [(64, 4096, -1, "uniform")])
    if name == "c3":
        return ("C3 mixed radix N in {60,105,210,1000,2187,3125}, batch=floor(2^26/N), fwd",
                [(n, ELEMS // n, -1, "uniform") for n in (60, 105, 210, 1000, 2187, 3125)])
    if name == "c5":
        return ("C5 distributed six-step N=2^30, one transform, block-distributed over the ranks, fwd",
                [(1 << 30, 1, -1, "uniform")])
    if name == "c4":
        return ("C4 four-step N in {2^16,2^20,2^24}, batch=2^28/N, fwd+inv",
                [(1 << k, (1 << 28) >> k, s, "normal") for k in (16, 20, 24) for s in (-1, 1)])
    raise ValueError(name)


def flops(N, batch):
    return 5.0 * N * math.log2(N) * batch if N > 1 else 0.0


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every 2 ms during the timed region."""

    def __init__(self, device_index=0, period=0.002):
        self.idx = device_index
        self.period = period
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None
        self.ok = False

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(self.idx).uuid)
                h = nv.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
            except Exception:
                h = nv.nvmlDeviceGetHandleByIndex(self.idx)
            bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                    "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                    "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
            self.mx.append(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.ok = True
            while True:
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                for name, b in bits.items():
                    if r & b:
                        self.reasons.add(name)
                if self._stop.wait(self.period):
                    break
            nv.nvmlShutdown()
        except Exception as e:  # pragma: no cover
            self.reasons.add("nvml unavailable: %s" % type(e).__name__)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.01)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ------------------------------------------------------------------ reference arm / cpu baseline
def oracle_run(jobs, budget_s=15.0, threads=0):
    """Time the oracle's O2 on a bounded sample of the workload.
    Returns (GFLOP/s, seconds, sample description, threads)."""
    import numpy as np
    import oracle
    import synth
    nthreads = threads or len(os.sched_getaffinity(0))
    # calibration: 2^16 elements of each job, scale the sample to the budget
    per = []
    for (N, batch, sign, dist) in jobs:
        nb = max(1, min(batch, (1 << 16) // N))
        x = synth.make(dist, N, nb, seed=0)
        t0 = time.perf_counter()
        oracle.fft_ct(x, sign, nthreads)
        per.append((time.perf_counter() - t0) / nb)
    tot_f, tot_t, parts = 0.0, 0.0, []
    for (N, batch, sign, dist), pt in zip(jobs, per):
        # equal time share per job
        nb = max(1, min(batch, int(budget_s / len(jobs) / max(pt, 1e-9))))
        x = synth.make(dist, N, nb, seed=0)
        t0 = time.perf_counter()
        oracle.fft_ct(x, sign, nthreads)
        dt = time.perf_counter() - t0
        tot_f += flops(N, nb)
        tot_t += dt
        parts.append("N=%d:%d" % (N, nb))
    return tot_f / tot_t / 1e9, tot_t, "transforms per job " + ",".join(parts), nthreads


# ------------------------------------------------------------------ fftc arm
def run_fftc(args):
    import torch
    import torch.distributed as dist
    import synth
    import paper_2207_06803_b200 as fftc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    desc, jobs = workloads(args.workload)

    # inputs: one buffer per distinct (element count, dist); rank r draws its own seeded batch
    bufs = {}
    for (N, batch, sign, d) in jobs:
        key = (N * batch, d, N if d == "normal" else 0)
        if key not in bufs:
            x = synth.make(d, N, batch, seed=synth.shard_seed(0, rank))
            xh = torch.from_numpy(x.reshape(-1)).pin_memory()
            bufs[key] = (xh, xh.to(dev))
    maxe = max(N * b for (N, b, _, _) in jobs)
    out = torch.empty(maxe, dtype=torch.complex64, device=dev)
    plans = [fftc.Plan(N, b, s) for (N, b, s, _) in jobs]
    launches_per_step = sum(p.launches() for p in plans)
    stream = torch.cuda.current_stream(dev)

    def one_step(evs=None):
        for i, ((N, b, s, d), p) in enumerate(zip(jobs, plans)):
            x = bufs[(N * b, d, N if d == "normal" else 0)][1]
            p.execute(x, out)
            if evs is not None:
                evs[i + 1].record(stream)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize(dev)

    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(jobs) + 1)] for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # inputs smaller than the 126 MB L2 (C1: 2 MiB) would stay L2-resident from step to step:
    # flush L2 between timed steps (a 256 MiB memset outside the per-step event pairs, which are
    # what is summed); larger inputs stream through HBM anyway
    in_bytes = sum(v[1].numel() * 8 for v in bufs.values())
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev) if in_bytes < (256 << 20) else None
    l2_note = ("inputs %.1f MiB < 126 MB L2: L2 flushed between timed steps (256 MiB memset outside "
               "the per-step events)" % (in_bytes / 2**20) if flush is not None
               else "inputs %d MiB > 126 MB L2, no flush" % (in_bytes >> 20))
    sampler = ClockSampler(local)
    with sampler:
        for k in range(K):
            if flush is not None:
                flush.zero_()
            evs[k][0].record(stream)
            one_step(evs[k])
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    step_ms = [evs[k][0].elapsed_time(evs[k][-1]) for k in range(K)]
    launch_ms = [[evs[k][i].elapsed_time(evs[k][i + 1]) for i in range(len(jobs))] for k in range(K)]
    t_rank = sum(step_ms) / 1e3
    if world > 1:
        tt = torch.tensor([t_rank], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = tt.item()
    else:
        t_max = t_rank
    step_flops = sum(flops(N, b) for (N, b, _, _) in jobs)
    value = world * K * step_flops / t_max / 1e9

    # per-job numbers (rank-local, mean over steps)
    per_job = []
    for i, (N, b, s, d) in enumerate(jobs):
        ts = sorted(launch_ms[k][i] / 1e3 for k in range(K))
        t = statistics.mean(ts)
        passes = plans[i].launches() if N > 4096 else 1  # HBM round trips (one per pass kernel)
        per_job.append({"N": N, "batch": b, "sign": s, "us": round(t * 1e6, 2),
                        "us_median": round(ts[len(ts) // 2] * 1e6, 2), "us_min": round(ts[0] * 1e6, 2),
                        "us_p90": round(ts[min(len(ts) - 1, int(0.9 * len(ts)))] * 1e6, 2),
                        "gflops": round(flops(N, b) / t / 1e9, 1),
                        "eff_GBs": round(16 * N * b / t / 1e9, 1), "hbm_passes": passes,
                        "plan": plans[i].describe()})

    # roofline of the dominant kernel family: the fused single-pass kernel (jobs with N <= 4096)
    # or, for large-N workloads, the TMA pass kernels (16 B per element per HBM pass)
    peak, peak_kind = measured_peaks()
    sp = [i for i, (N, b, s, d) in enumerate(jobs) if N <= 4096]
    large = not sp
    if large:
        sp = list(range(len(jobs)))
    rl = None
    if sp:
        t_mean = statistics.mean(launch_ms[k][i] for k in range(K) for i in sp) / 1e3
        bytes_mean = statistics.mean(16.0 * jobs[i][0] * jobs[i][1] * per_job[i]["hbm_passes"] for i in sp)
        ach = bytes_mean / t_mean / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic_%s.json" % args.workload)
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get("dram_bytes_per_launch")
        rl = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
              "frac": round(ach / peak, 4), "traffic": traffic,
              "kernel": ("k_pass (TMA tensor-tile Stockham pass, one launch per pass)" if large else
                         "k_fused_batch (fused Stockham, one launch per transform set)"),
              "algorithmic_bytes_per_launch": (bytes_mean / statistics.mean(per_job[i]["hbm_passes"] for i in sp)
                                               if large else bytes_mean),
              "peak_source": peak_kind}
    clocks = sampler.summary()

    # launch-latency-bound workloads: the same step captured in a CUDA graph (reps steps per replay)
    graph = None
    if args.graph or args.workload == "c1":
        reps = 50
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            one_step()  # warm on the capture stream
            torch.cuda.synchronize(dev)
            with torch.cuda.graph(g, stream=side):
                for _ in range(reps):
                    one_step()
        torch.cuda.synchronize(dev)
        g.replay()
        torch.cuda.synchronize(dev)
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ga.record(stream)
        for _ in range(K):
            g.replay()
        gb.record(stream)
        torch.cuda.synchronize(dev)
        gt = ga.elapsed_time(gb) / 1e3 / (K * reps)
        graph = {"ms_per_step": round(gt * 1e3, 5), "value": round(step_flops / gt / 1e9, 2), "unit": UNIT,
                 "steps_per_graph": reps,
                 "note": "CUDA graph replay of %d steps; device time per step%s" %
                         (reps, "; inputs L2-resident across the replayed steps" if flush is not None else "")}

    # e2e through the C ABI on host buffers (pinned), H2D + kernels + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        outs_h = torch.empty(maxe, dtype=torch.complex64).pin_memory()
        for (N, b, s, d), p in zip(jobs, plans):  # warm the staging buffers
            p.execute_host(bufs[(N * b, d, N if d == "normal" else 0)][0], outs_h)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        ke = max(1, min(K, 2))
        for _ in range(ke):
            for (N, b, s, d), p in zip(jobs, plans):
                p.execute_host(bufs[(N * b, d, N if d == "normal" else 0)][0], outs_h)
        te = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = tt.item()
        nbytes = sum(8 * N * b for (N, b, _, _) in jobs)
        e2e = {"value": round(world * ke * step_flops / te / 1e9, 2), "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "note": "fftc_execute_host, pinned host buffers, 32 MiB chunks over 3 streams"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, t, sample, th = oracle_run(jobs, budget_s=args.cpu_budget)
        cpu = {"value": round(v, 4), "unit": UNIT, "cores": th, "kind": "oracle",
               "sample": "O2 recursive Cooley-Tukey fp64 (oracle/oracle.c), %s; %.1f s" % (sample, t)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": round(t_max * 1e3 / K, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (complex64)",
            "data": "synthetic: re/im U[-1,1) (normal for C4), numpy PCG64 seed 0 (rank r: SeedSequence [0,r])",
            "config": {"workload": desc, "elements_per_transform_set": maxe,
                       "transform_sets_per_step": len(jobs), "l2": l2_note,
                       "parallelism": "batch-sharded weak scaling x%d" % world},
            "roofline": rl, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * K,
            "clocks": clocks, "per_job": per_job,
        }
        if graph:
            line["graph"] = graph
        print(json.dumps(line), flush=True)
    for p in plans:
        p.close()
    if world > 1:
        dist.destroy_process_group()


def run_c5(args):
    """Six-step over WORLD_SIZE ranks (NCCL all-to-alls); one rank = the same six-step on one GPU."""
    import torch
    import torch.distributed as dist
    import synth
    import paper_2207_06803_b200 as fftc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    N = args.c5_n
    if world > 1:
        dist.init_process_group("nccl")
        idt = torch.zeros(fftc.FFTC_NCCL_ID_BYTES, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(fftc.fftc_dist_get_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nid = bytes(idt.cpu().numpy().tobytes())
    else:
        nid = None
    lb = args.c5_loopback if world == 1 else 0
    plan = fftc.Plan.dist(N, -1, nid, rank, lb or world, loopback=bool(lb), flags=args.c5_flags)
    slab = N // world
    # rank r holds elements [r N/P, (r+1) N/P) of one seeded U[-1,1) vector (generated per slab
    # from a per-rank seed so no rank materialises the whole 8 GiB vector)
    x = torch.from_numpy(synth.uniform_c64(slab, 1, seed=synth.shard_seed(0, rank))[0]).to(dev)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        plan.execute(x, y)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    K = args.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        e0.record(stream)
        for _ in range(K):
            plan.execute(x, y)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    t = e0.elapsed_time(e1) / 1e3
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = tt.item()
    value = K * flops(N, 1) / t / 1e9
    if rank == 0:
        a2a_bytes = 3 * (world - 1) / world * 8 * N / world if world > 1 else 0
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": K,
                "warmup": args.warmup, "ms_per_step": round(t * 1e3 / K, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32 (complex64)",
                "data": "synthetic U[-1,1), per-rank seeded slabs",
                "config": {"workload": ("C5 six-step N=%d, %d virtual ranks on one GPU (loopback: the three "
                                        "all-to-alls are device copies)" % (N, lb)) if lb else
                                       ("C5 six-step N=%d over %d rank(s)" % (N, world)),
                           "plan": plan.describe(),
                           "nvlink_bytes_per_rank_per_step": a2a_bytes},
                "gpu_launches": plan.launches() * K, "clocks": sampler.summary()}
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    desc, jobs = workloads(args.workload)
    # each step: a bounded sample of the workload on the host cores (oracle as it stands)
    for _ in range(args.warmup):
        oracle_run(jobs[:1], budget_s=0.2)
    vals, ts, sample, th = [], 0.0, "", 0
    for _ in range(args.steps):
        v, t, sample, th = oracle_run(jobs, budget_s=min(args.ref_budget, 150.0 / max(1, args.steps)))
        vals.append(v)
        ts += t
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ts * 1e3 / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic, same seeds as the fftc arm",
            "config": {"workload": desc, "sample": sample},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": th, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fftc", choices=["fftc", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--c5-n", type=int, default=1 << 30)
    ap.add_argument("--c5-loopback", type=int, default=0,
                    help="one GPU: run the six-step for P virtual ranks (all-to-alls = device copies)")
    ap.add_argument("--c5-flags", type=int, default=0,
                    help="six-step options: 1 = transposed output (no all-to-all #3), 2 = fused peer-store exchanges")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true", help="also time the step captured in a CUDA graph")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "fftc":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c5":
        run_c5(args)
    else:
        run_fftc(args)


if __name__ == "__main__":
    main()
