"""Quick per-size kernel timing (CUDA events, L2 flushed between reps). Dev tool."""
import sys, json, math, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2207_06803_b200 as fftc

def bench(N, batch, sign=-1, reps=10):
    x = torch.randn(N * batch, dtype=torch.complex64, device="cuda")
    y = torch.empty_like(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    p = fftc.Plan(N, batch, sign)
    for _ in range(3):
        p.execute(x, y)
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); p.execute(x, y); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort(); t = ts[len(ts) // 2]
    passes = 2 if N > 4096 else 1
    gbs = 16 * N * batch / t / 1e9
    gflops = 5 * N * math.log2(N) * batch / t / 1e9
    return dict(N=N, batch=batch, sign=sign, us=t * 1e6, eff_GBs=gbs, hbm_GBs=gbs * passes, gflops=gflops,
                frac=gbs * passes / 6533.2, plan=p.describe())

sizes = [(1 << k, (1 << 26) >> k) for k in range(3, 13)] + [(n, (1 << 26) // n) for n in [60, 105, 210, 1000, 2187, 3125]] \
      + [(1 << k, (1 << 28) >> k) for k in (16, 20, 24)]
for N, b in sizes:
    r = bench(N, b)
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
