"""Run each given size once (after one warm-up) -- target for ncu --set full.  Dev tool.
    python tools/prof_one.py 128 2048 60 1048576 ...   (batch = 2^26/N, or 2^28/N above 4096)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2207_06803_b200 as fftc
for a in sys.argv[1:]:
    N = int(a)
    batch = ((1 << 28) if N > 4096 else (1 << 26)) // N
    x = torch.randn(N * batch, dtype=torch.complex64, device="cuda")
    y = torch.empty_like(x)
    with fftc.Plan(N, batch, -1) as p:
        p.execute(x, y)
        torch.cuda.synchronize()
        p.execute(x, y)
        torch.cuda.synchronize()
    del x, y
