"""A/B of large-N pass configurations on one GPU (dev tool).

    python tools/pass_ab.py N "label:ENV=VAL;ENV=VAL" "label2:..." ...

Each variant's plan is made with its environment (FFTC_PASS, FFTC_PASS_LOGS, ...), checked once
against numpy's fp64 FFT on two transforms (rel L2), then all variants are timed in alternating
rounds (CUDA events, batch = 2^26 / N up to 4096 else 2^28 / N, median ms; frac_copy_peak = one
HBM round trip (16 B per element) against the measured 6557 GB/s).  JSON line per variant."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_06803_b200 as fftc  # noqa: E402


def make(N, batch, sign, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fftc.Plan(N, batch, sign)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    N = int(sys.argv[1])
    variants = []
    for a in sys.argv[2:]:
        label, _, rest = a.partition(":")
        env = dict(kv.split("=", 1) for kv in rest.split(";") if kv)
        variants.append((label, env))
    batch = max(1, ((1 << 26) if N <= 4096 else (1 << 28)) // N)  # the BASELINE configs' sizes
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(batch, N, dtype=torch.complex64, device="cuda", generator=g)
    y = torch.empty_like(x)
    rounds = int(os.environ.get("ROUNDS", "5"))
    plans = []
    parity = os.environ.get("PARITY", "1") != "0"  # PARITY=0: timing only (very large N)
    xs = x[:2].cpu().numpy().astype(np.complex128) if parity else None
    for label, env in variants:
        rec = {"N": N, "label": label, "env": env}
        for sign in (-1, 1):
            p = make(N, batch, sign, env)
            p.execute(x, y)
            torch.cuda.synchronize()
            if parity:
                ref = np.fft.fft(xs, axis=1) if sign < 0 else np.fft.ifft(xs, axis=1) * N
                got = y[:2].cpu().numpy().astype(np.complex128)
                err = float((np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)).max())
                rec["rel_l2_%+d" % sign] = err
            if sign < 0:
                rec["plan"] = p.describe()
                plans.append((rec, p))
            else:
                p.close()
    times = {id(r): [] for r, _ in plans}
    for _ in range(rounds):
        for rec, p in plans:
            for _ in range(2):
                p.execute(x, y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(5):
                e0.record()
                p.execute(x, y)
                e1.record()
                e1.synchronize()
                times[id(rec)].append(e0.elapsed_time(e1))
    for rec, p in plans:
        ts = sorted(times[id(rec)])
        rec["ms_median"] = round(ts[len(ts) // 2], 4)
        rec["ms_min"] = round(ts[0], 4)
        rec["ms_per_2^28"] = round(rec["ms_median"] * (1 << 28) / (N * batch), 4)
        rec["frac_copy_peak"] = round(16.0 * N * batch / (rec["ms_median"] * 1e-3) / 6556.8e9, 4)
        print(json.dumps(rec), flush=True)
        p.close()


if __name__ == "__main__":
    main()
