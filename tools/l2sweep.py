"""Dev tool: time the L2-resident path for large N over env-tunable chunk sizes / grids."""
import os, sys, itertools, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "one":
    import torch, paper_2207_06803_b200 as fftc
    n, b = int(sys.argv[2]), int(sys.argv[3])
    N = 1 << n
    x = torch.randn(N * b, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
    p = fftc.Plan(N, b, -1)
    for _ in range(3): p.execute(x, y)
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        a.record(); p.execute(x, y); e.record(); e.synchronize(); ts.append(a.elapsed_time(e))
    ts.sort()
    print(json.dumps({"n": n, "b": b, "ms": round(ts[5], 4), "GBs": round(16 * N * b / ts[5] / 1e6, 1),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("FFTC_")}, "plan": p.describe()}), flush=True)
    sys.exit(0)
cases = [(16, 4096), (20, 256)]
for (n, b) in cases:
    for ch in os.environ.get("CHUNKS", "4,8,16,32").split(","):
        for grid in os.environ.get("GRIDS", "0").split(","):
            env = dict(os.environ, FFTC_L2_CHUNK_MB=ch)
            if grid != "0": env["FFTC_L2_GRID"] = grid
            subprocess.run([sys.executable, __file__, "one", str(n), str(b)], env=env, timeout=120)
