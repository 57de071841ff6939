"""PCIe / host-staging measurements for the e2e path (dev tool).
    python tools/host_bw.py            # JSON lines: raw H2D, D2H, both; execute_host per chunk/depth"""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

nbytes = 512 << 20
h_in = torch.empty(nbytes // 8, dtype=torch.complex64).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
d = torch.empty(nbytes // 8, dtype=torch.complex64, device="cuda")
d2 = torch.empty_like(d)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    d.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d2, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d2, non_blocking=True)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    t = timed(fn)
    print(json.dumps({"copy": name, "GBs_per_dir": round(nbytes / t / 1e9, 1)}), flush=True)

code = r'''
import sys, time, json, torch
sys.path.insert(0, ".")
import paper_2207_06803_b200 as fftc
N = 1024; batch = (512 << 20) // 8 // N
x = torch.randn(N * batch, dtype=torch.complex64).pin_memory(); y = torch.empty_like(x).pin_memory()
with fftc.Plan(N, batch, -1) as p:
    p.execute_host(x, y)
    t = time.perf_counter()
    for _ in range(5): p.execute_host(x, y)
    t = (time.perf_counter() - t) / 5
print(json.dumps({"chunk_mb": %s, "depth": %s, "ms": round(t * 1e3, 2), "GBs_per_dir": round((512 << 20) / t / 1e9, 1)}))
'''
for mb in (8, 32, 64, 128):
    for depth in (2, 3, 4):
        env = dict(os.environ, FFTC_HOST_CHUNK_MB=str(mb), FFTC_HOST_DEPTH=str(depth))
        r = subprocess.run([sys.executable, "-c", code % (mb, depth)], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-300:], flush=True)
