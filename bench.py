#!/usr/bin/env python3
"""bench.py -- batched 1D C2C FFT on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fftc|reference]
                    [--workload c2|c1|c3|c4|c5] [--no-extras]

Workload (default, BASELINE.json configs[1]): the power-of-two sweep
N = 2^3 ... 2^12, batch = 2^26/N (2^26 complex64 = 512 MiB per buffer), values
U[-1,1) from seed 0, forward AND inverse.  One step = the whole sweep = 20
fftc_execute calls (10 sizes x 2 signs), each a full pass of the hot path
(stage-in, Stockham stages, stage-out).

--gpus N: one process per GPU.  Without a torchrun environment bench.py launches
itself under torch.distributed.run.  The batch of every job is partitioned into
contiguous shards, rank r transforming [floor(rB/N), floor((r+1)B/N)) of the same
seeded input (drawn with PCG64.advance, bit-identical to those rows of the 1-GPU
input): strong scaling, no data-path collective.

value  = 5 N log2(N) flops of the whole job (all ranks) / max-over-ranks device time
         (CUDA events on the launch stream), GFLOP/s; value_std = std dev of the per-step
         values (one step = one round of the paper's protocol).
e2e    = the same metric through fftc_execute_host: pinned host input -> device ->
         transform -> host output, copies inside the timed region.
roofline: the dominant kernel (the fused Stockham kernel for C2/C3; the pass kernels for
         C4); achieved = SURVEY §8(d) algorithmic bytes (16 B per element, single pass;
         32 B per element for the C4 two-pass bound) / launch time.
c3 / c4: compact sub-records (N = 1) timing the mixed-radix and large-N configs beside
         the headline, each job's fraction of its §8(d) bound.
c5:    (N > 1) the distributed six-step N = 2^30 over the N ranks (NCCL all-to-alls; fused
         peer-store exchanges; fused + transposed output), run as its own torchrun job so a
         crash or hang there cannot cost the headline line.
cpu_baseline: the oracle's recursive Cooley-Tukey (oracle/, fp64, OpenMP) on a bounded
         sample of the same workload (rank 0, N = 1 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
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
L2_BYTES = 126 * 1000 * 1000
NOMINAL_HBM_GBS = 8000.0


def workloads(name):
    """-> (description, [(N, global batch, sign, dist)])"""
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
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def ncu_jobs(workload):
    """Per-job ncu numbers (gpu__time_duration, DRAM bytes) from the committed launch list
    (tools/ncu_jobs.py parse) -> {(N, sign): {...}} or {}."""
    p = os.path.join(ROOT, "profiles", "ncu_jobs_%s.json" % workload)
    if not os.path.exists(p):
        return {}, None
    d = json.load(open(p))
    return {(j["N"], j["sign"]): j for j in d["jobs"]}, d.get("source")


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every 2 ms during the timed region."""

    def __init__(self, device_index=0, period=0.002):
        self.idx = device_index
        self.period = period
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None

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


# ------------------------------------------------------------------ distributed helpers
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self):
        import torch
        # FFTC_BENCH_BACKEND=gloo (test only): several ranks may then share one GPU to exercise
        # the multi-rank logic on a one-GPU box (ranks never wait on one another's kernels)
        backend = os.environ.get("FFTC_BENCH_BACKEND", "nccl")
        if backend != "nccl":
            self.local = self.local % torch.cuda.device_count()
        torch.cuda.set_device(self.local)
        if self.world > 1:
            import torch.distributed as dist
            import datetime
            # long timeout: ranks != 0 wait at a barrier while rank 0 runs the c5 child job
            kw = {"device_id": torch.device("cuda", self.local)} if backend == "nccl" else {}
            dist.init_process_group(backend, timeout=datetime.timedelta(minutes=30), **kw)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, values):
        """elementwise max over ranks of a list of floats"""
        if not self.pg:
            return list(values)
        import torch
        nccl = os.environ.get("FFTC_BENCH_BACKEND", "nccl") == "nccl"
        t = torch.tensor(list(values), dtype=torch.float64, device="cuda" if nccl else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return t.tolist()

    def gather_strings(self, s):
        if not self.pg:
            return [s]
        out = [None] * self.world
        self.pg.all_gather_object(out, s)
        return out

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ------------------------------------------------------------------ fftc arm
class JobSet:
    """Plans + device buffers for one workload on this rank (its batch shard of every job)."""

    def __init__(self, jobs, dev, rank, world):
        import torch
        import synth
        import paper_2207_06803_b200 as fftc
        self.dev = dev
        self.jobs = []  # (N, global batch, sign, dist, b0, b1)
        for (N, B, s, d) in jobs:
            b0, b1 = synth.shard_range(B, rank, world)
            self.jobs.append((N, B, s, d, b0, b1))
        # inputs: uniform jobs read elements [N b0, N b1) of the one seeded stream; drawn once as
        # the union of the ranges, each job gets its own 16-byte aligned device copy of its range
        self.host = {}
        uni = [(N * b0, N * b1) for (N, B, s, d, b0, b1) in self.jobs if d == "uniform"]
        stream = None
        if uni:
            E0, E1 = min(a for a, _ in uni), max(b for _, b in uni)
            stream = synth.uniform_c64_rows(1, E0, E1, seed=0).reshape(-1)
        self.keys, dbufs = [], {}
        for (N, B, s, d, b0, b1) in self.jobs:
            if d == "uniform":
                key = ("u", N * b0, N * b1)
                if key not in self.host:
                    self.host[key] = torch.from_numpy(stream[N * b0 - E0:N * b1 - E0]).pin_memory()
            else:  # standard normal: not sliceable by advance (single GPU only); the flat stream
                if world != 1:  # of normal_c64(N, B) does not depend on N, so sizes share it
                    raise SystemExit("normal-distributed workloads (C4) are single-GPU")
                key = ("n", N * B)
                if key not in self.host:
                    self.host[key] = torch.from_numpy(synth.normal_c64(N * B, 1, seed=0).reshape(-1)).pin_memory()
            self.keys.append(key)
        # rotation: when one job's in + out (this rank's shard) is small against the L2, several
        # copies of the input and output are cycled so no job reads data a previous job left in L2
        per_job = max((N * (b1 - b0) * 8 for (N, B, s, d, b0, b1) in self.jobs), default=0)
        self.nrot = 1 if per_job == 0 else max(1, math.ceil(3 * L2_BYTES / (2 * per_job)))
        self.flush = None
        if self.nrot > 16:  # tiny inputs (C1): flush L2 between steps instead
            self.nrot = 1
            self.flush = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
        for key, h in self.host.items():
            d0 = h.to(dev)
            dbufs[key] = [d0] + [d0.clone() for _ in range(self.nrot - 1)]
        self.dbufs = dbufs
        maxe = max([N * (b1 - b0) for (N, B, s, d, b0, b1) in self.jobs] + [1])
        self.outs = [torch.empty(maxe, dtype=torch.complex64, device=dev) for _ in range(self.nrot)]
        self.plans = [fftc.Plan(N, b1 - b0, s) for (N, B, s, d, b0, b1) in self.jobs]
        self.maxe = maxe
        self.cursor = 0

    def launches(self):
        return sum(p.launches() for p in self.plans)

    def run(self, stream, evs=None):
        for i, p in enumerate(self.plans):
            r = self.cursor % self.nrot
            self.cursor += 1
            p.execute(self.dbufs[self.keys[i]][r], self.outs[r])
            if evs is not None:
                evs[i + 1].record(stream)

    def l2_note(self):
        if self.flush is not None:
            return "inputs < L2: L2 flushed between timed steps (a 256 MiB read sweep outside the per-step events)"
        if self.nrot > 1:
            return ("per-rank buffers small against the 126 MB L2: %d input/output copies rotated so "
                    "every launch reads data no recent launch touched" % self.nrot)
        return "inputs larger than the 126 MB L2 (each launch streams >= 2x L2), no flush"

    def close(self):
        for p in self.plans:
            p.close()


def time_jobset(js, dev, K, W, dist_=None, sampler=None):
    """W warm-up steps, then K timed steps; per-step and per-launch CUDA-event times (s)."""
    import torch
    stream = torch.cuda.current_stream(dev)
    for _ in range(W):
        js.run(stream)
    torch.cuda.synchronize(dev)
    n = len(js.plans)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(K)]
    if dist_:
        dist_.barrier()
    torch.cuda.synchronize(dev)
    ctx = sampler if sampler is not None else _Null()
    with ctx:
        for k in range(K):
            if js.flush is not None:
                js.flush.sum()  # a read-only sweep: evicts the inputs without leaving dirty lines to write back
            evs[k][0].record(stream)
            js.run(stream, evs[k])
        torch.cuda.synchronize(dev)
    if dist_:
        dist_.barrier()
    step = [evs[k][0].elapsed_time(evs[k][-1]) / 1e3 for k in range(K)]
    launch = [[evs[k][i].elapsed_time(evs[k][i + 1]) / 1e3 for i in range(n)] for k in range(K)]
    return step, launch


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def per_job_records(js, launch, K, ncu=None, peak=None):
    out = []
    for i, (N, B, s, d, b0, b1) in enumerate(js.jobs):
        b = b1 - b0
        ts = sorted(launch[k][i] for k in range(K))
        t = statistics.mean(ts)
        passes = js.plans[i].launches() if N > 4096 else 1  # HBM round trips (one per pass kernel)
        r = {"N": N, "batch": b, "sign": s, "us": round(t * 1e6, 2),
             "us_median": round(ts[len(ts) // 2] * 1e6, 2), "us_min": round(ts[0] * 1e6, 2),
             "us_p90": round(ts[min(len(ts) - 1, int(0.9 * len(ts)))] * 1e6, 2),
             "us_std": round(statistics.pstdev(ts) * 1e6, 2),
             "gflops": round(flops(N, b) / t / 1e9, 1),
             "eff_GBs": round(16 * N * b / t / 1e9, 1), "hbm_passes": passes,
             "plan": js.plans[i].describe()}
        if ncu and (N, s) in ncu:
            j = ncu[(N, s)]
            r["ncu_us"] = j["us"]
            r["ncu_dram_GBs"] = j["dram_GBs"]
            r["ncu_dram_bytes_per_elt"] = j["dram_bytes_per_elt"]
            r["pct_peak_measured"] = round(100 * j["dram_GBs"] / peak, 1)
            r["pct_peak_nominal"] = round(100 * j["dram_GBs"] / NOMINAL_HBM_GBS, 1)
        out.append(r)
    return out


def sub_record(workload, dev, K, W, peak):
    """Compact timing of another config on this GPU (N = 1): per size mean us and the fraction
    of its SURVEY §8(d) bound (C3: 16 B/element; C4: 32 B/element, the two-pass bound)."""
    desc, jobs = workloads(workload)
    js = JobSet(jobs, dev, 0, 1)
    step, launch = time_jobset(js, dev, K, W)
    ncu, src = ncu_jobs(workload)
    rows = per_job_records(js, launch, K, ncu, peak)
    bpe = 32.0 if workload == "c4" else 16.0
    recs = []
    for r in rows:
        e = r["N"] * r["batch"]
        rec = {"N": r["N"], "sign": r["sign"], "us": r["us"], "us_std": r["us_std"], "gflops": r["gflops"],
               "hbm_passes": r["hbm_passes"],
               "frac": round(bpe * e / (r["us"] * 1e-6) / 1e9 / peak, 4)}
        if workload == "c4":
            rec["ms_per_2^28_elts"] = round(r["us"] / 1e3 * (1 << 28) / e, 4)
            rec["frac_impl_passes"] = round(16.0 * r["hbm_passes"] * e / (r["us"] * 1e-6) / 1e9 / peak, 4)
        for k in ("ncu_dram_GBs", "ncu_dram_bytes_per_elt", "pct_peak_measured", "pct_peak_nominal"):
            if k in r:
                rec[k] = r[k]
        recs.append(rec)
    tot = sum(step)
    val = K * sum(flops(N, B) for (N, B, s, d) in jobs) / tot / 1e9
    js.close()
    import torch
    torch.cuda.empty_cache()
    return {"workload": desc, "value": round(val, 1), "unit": UNIT, "steps": K, "warmup": W,
            "bound_bytes_per_elt": bpe, "frac_min": min(r["frac"] for r in recs),
            "ncu_source": src, "jobs": recs}


def c5_child(args, world):
    """The distributed six-step at N = 2^30 over `world` ranks, run as a SEPARATE torchrun job
    (rank 0 of the headline run launches it and waits, the other ranks wait at a barrier), so a
    crash or hang in the NCCL / CUDA-IPC exchanges -- code that has not run on real NVLink yet --
    cannot cost the headline line.  Returns the child's JSON record or {"error": ...}."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "GROUP_RANK", "ROLE_RANK",
                        "ROLE_WORLD_SIZE", "GROUP_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT")
           and not k.startswith("TORCHELASTIC")}
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           "--gpus", str(world), "--workload", "c5", "--steps", "5", "--warmup", "2", "--c5-variants", "0,2,3"]
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=args.c5_timeout)
    except subprocess.TimeoutExpired:
        return {"error": "six-step child job not finished after %d s" % args.c5_timeout}
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    if r.returncode != 0 or not lines:
        # the ranks' own error lines (torchrun's summary at the end of stderr names no cause)
        out = (r.stderr or "") + (r.stdout or "")
        cause = [ln.strip() for ln in out.splitlines()
                 if any(w in ln for w in ("Error", "error:", "FFTC_", "NCCL WARN", "what():"))
                 and "elastic" not in ln and "errors.html" not in ln]
        return {"error": "six-step child job rc=%d: %s" % (r.returncode, " | ".join(cause[-4:]) or out[-400:])}
    d = json.loads(lines[-1])
    return {k: d[k] for k in ("value", "unit", "ms_per_step", "n_gpus", "variants", "a2a_reference", "config") if k in d}


def run_fftc(args):
    import torch
    import paper_2207_06803_b200 as fftc

    D = Dist()
    if D.world != args.gpus:
        raise SystemExit("bench.py: WORLD_SIZE=%d but --gpus %d" % (D.world, args.gpus))
    D.init()
    dev = torch.device("cuda", D.local)
    desc, jobs = workloads(args.workload)
    js = JobSet(jobs, dev, D.rank, D.world)
    launches_per_step = js.launches()
    K, W = args.steps, args.warmup
    sampler = ClockSampler(D.local)
    step, launch = time_jobset(js, dev, K, W, D, sampler)
    step_max = D.max(step)  # per step, max over ranks
    t_max = D.max([sum(step)])[0]
    step_flops = sum(flops(N, B) for (N, B, s, d) in jobs)  # whole job, all ranks
    value = K * step_flops / t_max / 1e9
    step_vals = [step_flops / t / 1e9 for t in step_max]
    peak, peak_kind = measured_peaks()
    ncu, ncu_src = ncu_jobs(args.workload) if D.world == 1 else ({}, None)
    per_job = per_job_records(js, launch, K, ncu, peak)

    # roofline of the dominant kernel: the fused single-pass kernel (every C1/C2/C3 launch is one);
    # for C4 the TMA pass kernels, against the §8(d) two-pass bound (32 B per element per job)
    large = all(N > 4096 for (N, B, s, d) in jobs)
    bpe = 32.0 if large else 16.0
    elts = [N * (b1 - b0) for (N, B, s, d, b0, b1) in js.jobs]
    t_job = statistics.mean(launch[k][i] for k in range(K) for i in range(len(jobs)))
    ach = statistics.mean(bpe * e for e in elts) / t_job / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic_%s.json" % args.workload)
    if os.path.exists(tf) and D.world == 1:
        traffic = json.load(open(tf)).get("dram_bytes_per_launch")
    rl = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
          "frac": round(ach / peak, 4), "traffic": traffic,
          "kernel": ("k_pass (TMA tensor-tile Stockham passes; bound = SURVEY §8(d) two-pass 32 B/element)"
                     if large else "k_fused_batch (fused Stockham, one launch per transform set)"),
          "algorithmic_bytes_per_launch": (None if large else statistics.mean(16.0 * e for e in elts)),
          "algorithmic_bytes_per_job": statistics.mean(bpe * e for e in elts),
          "peak_source": peak_kind}
    clocks = sampler.summary()

    graph = None
    if args.graph or args.workload == "c1":
        graph = time_graph(js, dev, K, step_flops / D.world)

    e2e = None
    if not args.no_e2e:
        e2e = time_e2e(js, D, K, step_flops)

    topo = None
    if D.world > 1:
        uuids = D.gather_strings(str(torch.cuda.get_device_properties(dev).uuid))
        topo = {"comm_nranks_ok": len(uuids) == args.gpus, "gpus_active": len(set(uuids))}

    line_holder = {}
    if D.world == 1 and args.workload == "c2" and not args.no_extras:
        js.close()
        js.dbufs, js.outs = {}, []
        torch.cuda.empty_cache()
        for w in ("c3", "c4"):
            try:
                line_holder[w] = sub_record(w, dev, min(K, 10), 3, peak)
            except Exception as e:  # reported, never fatal for the headline line
                line_holder[w] = {"error": "%s: %s" % (type(e).__name__, e)}

    cpu = None
    if D.rank == 0 and D.world == 1 and not args.no_cpu:
        v, t, sample, th = oracle_run(jobs, budget_s=args.cpu_budget)
        cpu = {"value": round(v, 4), "unit": UNIT, "cores": th, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": "O2 recursive Cooley-Tukey fp64 (oracle/oracle.c), %s; %.1f s" % (sample, t)}

    def emit():
        if D.rank != 0:
            return
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": D.world, "steps": K,
            "warmup": W, "ms_per_step": round(t_max * 1e3 / K, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (complex64)",
            "value_std": round(statistics.pstdev(step_vals), 2), "rounds": K,
            "data": "synthetic: re/im U[-1,1) (normal for C4), numpy PCG64 seed 0; rank r transforms "
                    "its contiguous batch shard of the same stream (PCG64.advance)",
            "config": {"workload": desc, "elements_per_transform_set": ELEMS if args.workload in ("c2", "c3")
                       else max(N * B for (N, B, s, d) in jobs),
                       "transform_sets_per_step": len(jobs), "l2": js.l2_note(),
                       "parallelism": "batch shards x%d (contiguous partition, no data-path collective)" % D.world},
            "roofline": rl, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * K,
            "clocks": clocks, "per_job": per_job,
        }
        if ncu_src:
            line["ncu_source"] = ncu_src
        if topo:
            line["multi_gpu"] = topo
        if graph:
            line["graph"] = graph
        for k in ("c3", "c4", "c5"):
            if k in line_holder:
                line[k] = line_holder[k]
        print(json.dumps(line), flush=True)

    if D.world > 1 and args.workload == "c2" and not args.no_extras:
        # the six-step over NCCL / NVLink in its own job (c5_child); the ranks of this job free
        # their buffers and wait
        js.close()
        js.dbufs, js.outs = {}, []
        torch.cuda.empty_cache()
        if D.rank == 0:
            line_holder["c5"] = c5_child(args, D.world)
        D.barrier()
    emit()
    js.close()
    D.close()


def time_graph(js, dev, K, step_flops_rank):
    """Launch-latency-bound workloads: the step captured in a CUDA graph (reps steps per replay)."""
    import torch
    stream = torch.cuda.current_stream(dev)
    reps = 50
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        js.run(side)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(g, stream=side):
            for _ in range(reps):
                js.run(side)
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
    return {"ms_per_step": round(gt * 1e3, 5), "value": round(step_flops_rank / gt / 1e9, 2), "unit": UNIT,
            "steps_per_graph": reps,
            "note": "CUDA graph replay of %d steps; device time per step%s" %
                    (reps, "; inputs L2-resident across the replayed steps" if js.flush is not None else "")}


def time_e2e(js, D, K, step_flops):
    """The same metric through fftc_execute_host (the C ABI on pinned host buffers): H2D of the
    inputs, the kernels and D2H of the results inside the timed region."""
    import torch
    outs_h = torch.empty(js.maxe, dtype=torch.complex64).pin_memory()
    for i, p in enumerate(js.plans):  # warm the staging buffers
        p.execute_host(js.host[js.keys[i]], outs_h)
    D.barrier()
    t0 = time.perf_counter()
    ke = max(1, min(K, 2))
    for _ in range(ke):
        for i, p in enumerate(js.plans):
            p.execute_host(js.host[js.keys[i]], outs_h)
    te = D.max([time.perf_counter() - t0])[0]
    nbytes = sum(8 * N * (b1 - b0) for (N, B, s, d, b0, b1) in js.jobs)
    return {"value": round(ke * step_flops / te / 1e9, 2), "unit": UNIT,
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "note": "fftc_execute_host, pinned host buffers, 32 MiB chunks over 3 streams; per-rank bytes"}


def run_c5(args):
    """Six-step over WORLD_SIZE ranks (NCCL all-to-alls); one rank = the single-GPU plan."""
    import torch
    import synth
    import paper_2207_06803_b200 as fftc

    D = Dist()
    D.init()
    dev = torch.device("cuda", D.local)
    N = args.c5_n
    if D.world > 1:
        idt = torch.zeros(fftc.FFTC_NCCL_ID_BYTES, dtype=torch.uint8, device=dev)
        if D.rank == 0:
            idt.copy_(torch.frombuffer(bytearray(fftc.fftc_dist_get_unique_id()), dtype=torch.uint8))
        D.pg.broadcast(idt, 0)
        nid = bytes(idt.cpu().numpy().tobytes())
    else:
        nid = None
    lb = args.c5_loopback if D.world == 1 else 0
    if args.c5_variants:
        return run_c5_variants(args, D, dev, N)
    plan = fftc.Plan.dist(N, -1, nid, D.rank, lb or D.world, loopback=bool(lb), flags=args.c5_flags)
    slab = N // D.world
    # rank r holds elements [r N/P, (r+1) N/P) of the one seeded U[-1,1) vector
    x = torch.from_numpy(synth.uniform_c64_rows(1, D.rank * slab, (D.rank + 1) * slab, seed=0).reshape(-1)).to(dev)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        plan.execute(x, y)
    torch.cuda.synchronize(dev)
    D.barrier()
    K = args.steps
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    sampler = ClockSampler(D.local)
    with sampler:
        evs[0].record(stream)
        for k in range(K):
            plan.execute(x, y)
            evs[k + 1].record(stream)
        torch.cuda.synchronize(dev)
    steps = D.max([evs[k].elapsed_time(evs[k + 1]) / 1e3 for k in range(K)])
    t = D.max([evs[0].elapsed_time(evs[-1]) / 1e3])[0]
    value = K * flops(N, 1) / t / 1e9
    if D.rank == 0:
        a2a_bytes = 3 * (D.world - 1) / D.world * 8 * N / D.world if D.world > 1 else 0
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": D.world, "steps": K,
                "warmup": args.warmup, "ms_per_step": round(t * 1e3 / K, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32 (complex64)",
                "value_std": round(statistics.pstdev([flops(N, 1) / s / 1e9 for s in steps]), 2), "rounds": K,
                "data": "synthetic U[-1,1), rank r holds elements [rN/P,(r+1)N/P) of the seed-0 stream",
                "config": {"workload": ("C5 six-step N=%d, %d virtual ranks on one GPU (loopback: the three "
                                        "all-to-alls are device copies)" % (N, lb)) if lb else
                                       ("C5 six-step N=%d over %d rank(s)" % (N, D.world)),
                           "plan": plan.describe(),
                           "nvlink_bytes_per_rank_per_step": a2a_bytes},
                "gpu_launches": plan.launches() * K, "clocks": sampler.summary()}
        print(json.dumps(line), flush=True)
    plan.close()
    D.close()


def run_c5_variants(args, D, dev, N):
    """Six-step over the ranks for each exchange mode in --c5-variants (0: NCCL all-to-alls,
    2: fused peer stores, 3: fused + transposed output); one line with every variant's time."""
    import torch
    import synth
    import paper_2207_06803_b200 as fftc
    P = D.world
    slab = N // P
    x = torch.from_numpy(synth.uniform_c64_rows(1, D.rank * slab, (D.rank + 1) * slab, seed=0).reshape(-1)).to(dev)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    a2a = (P - 1) / P * 8 * N / P
    names = {0: "nccl a2a x3", 1: "nccl, transposed out", 2: "fused peer stores", 3: "fused peer stores + transposed out"}
    out = []
    for flags in [int(v) for v in args.c5_variants.split(",")]:
        idt = torch.zeros(fftc.FFTC_NCCL_ID_BYTES, dtype=torch.uint8, device=dev)
        if D.rank == 0:
            idt.copy_(torch.frombuffer(bytearray(fftc.fftc_dist_get_unique_id()), dtype=torch.uint8))
        D.pg.broadcast(idt, 0)
        plan = fftc.Plan.dist(N, -1, bytes(idt.cpu().numpy().tobytes()), D.rank, P, flags=flags)
        for _ in range(args.warmup):
            plan.execute(x, y)
        torch.cuda.synchronize(dev)
        D.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            plan.execute(x, y)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t = D.max([e0.elapsed_time(e1) / 1e3])[0] / args.steps
        na2a = 2 if flags & 1 else 3
        out.append({"flags": flags, "exchange": names.get(flags, str(flags)), "ms": round(t * 1e3, 3),
                    "gflops": round(flops(N, 1) / t / 1e9, 1), "a2a_per_step": na2a,
                    "nvlink_bytes_per_rank_per_a2a": a2a,
                    "nvlink_GBs_per_rank_lower_bound": round(na2a * a2a / t / 1e9, 1), "plan": plan.describe()})
        plan.close()
    # reference: torch.distributed all_to_all_single (NCCL) of the same 8N/P bytes per rank on the
    # same ranks -- the measured NVLink rate the six-step's exchanges are compared with
    ref = None
    try:
        src = x.view(torch.float32)
        dst = torch.empty_like(src)
        for _ in range(2):
            D.pg.all_to_all_single(dst, src)
        torch.cuda.synchronize(dev)
        D.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            D.pg.all_to_all_single(dst, src)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ta = D.max([e0.elapsed_time(e1) / 1e3])[0] / 5
        ref = {"ms": round(ta * 1e3, 3), "nvlink_GBs_per_rank": round(a2a / ta / 1e9, 1),
               "note": "torch.distributed.all_to_all_single of 8N/P bytes per rank, (P-1)/P of them over NVLink"}
    except Exception as e:  # reported, never fatal
        ref = {"error": "%s: %s" % (type(e).__name__, e)}
    if D.rank == 0:
        best = min(out, key=lambda v: v["ms"])
        print(json.dumps({"metric": METRIC, "value": best["gflops"], "unit": UNIT, "n_gpus": P,
                          "ms_per_step": best["ms"], "variants": out, "a2a_reference": ref,
                          "config": {"workload": "C5 six-step N=%d over %d ranks" % (N, P)}}), flush=True)
    D.close()


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
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "value_std": round(statistics.pstdev(vals), 4), "rounds": args.steps,
            "data": "synthetic, same seeds as the fftc arm",
            "config": {"workload": desc, "sample": sample},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": th, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def relaunch(args):
    """--gpus N without a torchrun environment: launch N ranks of this script under
    torch.distributed.run on this node (127.0.0.1) and return its exit code."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
    ap.add_argument("--c5-timeout", type=int, default=150, help="time limit of the c5 sub-record's job (N > 1)")
    ap.add_argument("--c5-variants", default="", help="--workload c5: time these exchange modes, e.g. 0,2,3")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the c3/c4 (N = 1) or c5 (N > 1) sub-records")
    ap.add_argument("--graph", action="store_true", help="also time the step captured in a CUDA graph")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=10.0)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
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
