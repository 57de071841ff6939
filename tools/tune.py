"""Time every compiled candidate schedule per N (FFTC_KERNEL=<name>), CUDA events, inputs > L2.
Dev tool; prints one JSON line per candidate.  python tools/tune.py [N ...]"""
import json, math, os, re, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2207_06803_b200 as fftc

sizes = [int(a) for a in sys.argv[1:]] or [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 60, 105, 210, 1000, 2187, 3125]
cands = {N: fftc.fftc_candidates(N) for N in sizes}
x = torch.randn(1 << 26, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
for N in sizes:
    batch = (1 << 26) // N
    for name in cands.get(N, []):
        os.environ["FFTC_KERNEL"] = name
        p = fftc.Plan(N, batch, -1)
        assert name in p.describe(), p.describe()
        for _ in range(3):
            p.execute(x, y)
        ts = []
        for _ in range(15):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); p.execute(x, y); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        ts.sort(); t = ts[len(ts) // 2]
        print(json.dumps({"N": N, "kernel": name, "us": round(t * 1e6, 1), "frac": round(16 * N * batch / t / 1e9 / 6533.2, 3)}), flush=True)
        p.close()
os.environ.pop("FFTC_KERNEL", None)
