"""Interleaved A/B timing of compiled single-pass candidates (FFTC_KERNEL=<name>) at a BASELINE size.

    python tools/ab_kernels.py N name1 name2 ... [--rounds 5] [--reps 15]

Every candidate gets its plan up front; rounds alternate between candidates so drift (clocks,
temperature) hits all of them alike.  Inputs are 2^26 complex64 (512 MiB > L2), uniform from
seed 0.  One JSON line per candidate: median and best-round median us, fraction of the measured
copy peak (16 B per element).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("N", type=int)
    ap.add_argument("names", nargs="*")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--sign", type=int, default=-1)
    a = ap.parse_args()
    import torch
    import paper_2207_06803_b200 as fftc
    import synth
    N = a.N
    batch = (1 << 26) // N
    names = a.names or fftc.fftc_candidates(N)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6556.8
    x = torch.from_numpy(synth.uniform_c64(N, batch, seed=0)).cuda()
    y = torch.empty_like(x)
    plans = {}
    for n in names:
        os.environ["FFTC_KERNEL"] = n
        p = fftc.Plan(N, batch, a.sign)
        if n not in p.describe():
            raise SystemExit("candidate %s not selected: %s" % (n, p.describe()))
        plans[n] = p
    os.environ.pop("FFTC_KERNEL", None)
    meds = {n: [] for n in names}
    for _ in range(a.rounds):
        for n, p in plans.items():
            for _ in range(3):
                p.execute(x, y)
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                p.execute(x, y)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            meds[n].append(statistics.median(ts))
    for n in names:
        m = statistics.median(meds[n])
        print(json.dumps({"N": N, "kernel": n, "us": round(m, 2), "us_best_round": round(min(meds[n]), 2),
                          "frac": round(16 * N * batch / (m * 1e-6) / 1e9 / peak, 4)}), flush=True)


if __name__ == "__main__":
    main()
