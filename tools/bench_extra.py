"""Measurements beyond the BASELINE configs (one GPU, CUDA events, median of 10).

    python tools/bench_extra.py > gpurun_out/extra.jsonl

Rows: the tensor-core direct DFT vs the Stockham kernel (N = 16, 32), JIT sizes, the
runtime-schedule passes for non-power-of-two large N, the L2-resident variant, the 8-CTA cluster
single pass for 2^16, 2^24 as two register-resident 4096-long passes, 2^22 / 2^23 (register 4096
first pass, the defaults), and the six-step in loopback mode (P virtual ranks on one GPU).  Effective GB/s counts 16 B per
element (one read + one write); `hbm_passes` says how often the data crosses HBM.
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_06803_b200 as fftc  # noqa: E402


def timed(p, x, y, reps=10):
    for _ in range(3):
        p.execute(x, y)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        p.execute(x, y)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


def row(tag, N, batch, p, t, passes=None):
    r = {"row": tag, "N": N, "batch": batch, "us": round(t * 1e6, 1),
         "gflops": round(5 * N * math.log2(N) * batch / t / 1e9, 1),
         "eff_GBs": round(16 * N * batch / t / 1e9, 1), "plan": p.describe()}
    if passes:
        r["hbm_passes"] = passes
        r["hbm_GBs"] = round(16 * N * batch * passes / t / 1e9, 1)
    print(json.dumps(r), flush=True)


def main():
    dev = torch.device("cuda", 0)
    x = torch.randn(1 << 26, dtype=torch.complex64, device=dev)
    y = torch.empty_like(x)
    for N in (16, 32):
        b = (1 << 26) // N
        for tag, mk in (("direct_tc", lambda: fftc.Plan.direct(N, b, -1)), ("stockham", lambda: fftc.Plan(N, b, -1))):
            p = mk()
            row(tag, N, b, p, timed(p, x, y), 1)
            p.close()
    for N in (11, 13, 61, 143, 3328):
        b = (1 << 26) // N
        p = fftc.Plan(N, b, -1)
        row("jit", N, b, p, timed(p, x, y), 1)
        p.close()
    del x, y
    x = torch.randn(1 << 28, dtype=torch.complex64, device=dev)
    y = torch.empty_like(x)
    for N in (59049, 100000, 10 ** 6):
        b = (1 << 28) // N
        p = fftc.Plan(N, b, -1)
        row("gpass", N, b, p, timed(p, x, y, 5), p.launches())
        p.close()
    os.environ["FFTC_LARGE"] = "l2"
    for N in (1 << 16, 1 << 20):
        b = (1 << 28) // N
        p = fftc.Plan(N, b, -1)
        row("l2_resident", N, b, p, timed(p, x, y, 5), 1)
        p.close()
    del os.environ["FFTC_LARGE"]
    for tag, N, env, passes in (("cluster_single_pass", 1 << 16, {"FFTC_LARGE": "cluster"}, 1),
                                ("register_4096_two_pass", 1 << 24,
                                 {"FFTC_PASS_LOGS": "12,12", "FFTC_PASS": "rp4096_r16x16x16_c4"}, 2),
                                ("default_2^22", 1 << 22, {}, 2), ("default_2^23", 1 << 23, {}, 2)):
        b = (1 << 28) // N
        os.environ.update(env)
        try:
            p = fftc.Plan(N, b, -1)
        finally:
            for k in env:
                del os.environ[k]
        row(tag, N, b, p, timed(p, x, y, 5), passes)
        p.close()
    del x, y
    torch.cuda.empty_cache()
    N = 1 << 30
    x = torch.randn(N, dtype=torch.complex64, device=dev)
    y = torch.empty_like(x)
    for P, flags in ((1, 0), (8, 0), (8, fftc.FFTC_DIST_PEER_STORES),
                     (8, fftc.FFTC_DIST_PEER_STORES | fftc.FFTC_DIST_TRANSPOSED_OUT)):
        p = fftc.Plan.dist(N, -1, None, 0, P, loopback=P > 1, flags=flags)
        row("six_step_loopback_P%d_flags%d" % (P, flags), N, 1, p, timed(p, x, y, 3))
        p.close()


if __name__ == "__main__":
    main()
