"""Median CUDA-event time per plan for the given sizes (batch = 2^26/N up to 4096, else max(1, 2^28/N)).
Dev tool for A/B of library builds: FFTC_LIB_PATH=<variant .so> python tools/time_sizes.py N ..."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2207_06803_b200 as fftc

tag = os.environ.get("TAG", os.path.basename(fftc.LIB_PATH))
sizes = [int(a) for a in sys.argv[1:]]
x = torch.randn(max([1 << 28] + sizes), dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
for N in sizes:
    batch = max(1, ((1 << 28) if N > 4096 else (1 << 26)) // N)
    with fftc.Plan(N, batch, -1) as p:
        for _ in range(3):
            p.execute(x, y)
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); p.execute(x, y); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(json.dumps({"tag": tag, "N": N, "ms": round(ts[5], 4), "plan": p.describe()[:80]}), flush=True)
