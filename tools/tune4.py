"""Tune the four-step: split M x K, column-pass and row-pass candidates (FFTC_SPLIT_M / FFTC_COL / FFTC_ROW).
Dev tool; JSON line per configuration.  python tools/tune4.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2207_06803_b200 as fftc

COLS = {256: ["c256_r16x16_t16x16", "c256_r16x16_t16x32", "c256_r16x16_t16x8"],
        512: ["c512_r16x32_t16x16", "c512_r32x16_t16x16", "c512_r32x16_t16x8"],
        1024: ["c1024_r32x32_t32x8", "c1024_r32x32_t32x4", "c1024_r32x32_t32x16", "c1024_r16x16x4_t64x8"],
        2048: ["c2048_r8x16x16_t128x4", "c2048_r16x16x8_t128x4", "c2048_r16x16x8_t128x2"],
        4096: ["c4096_r16x16x16_t256x4", "c4096_r16x16x16_t256x2", "c4096_r16x16x16_t128x4"]}
ROWS = {256: ["r256_r16x16_t16x32", "r256_r16x16_t16x16", "r256_r16x16_t16x8"],
        512: ["r512_r32x16_t16x16"],
        1024: ["r1024_r32x32_t32x8", "r1024_r32x32_t32x4", "r1024_r32x32_t32x16"],
        2048: ["r2048_r16x16x8_t128x4"],
        4096: ["r4096_r16x16x16_t256x4", "r4096_r16x16x16_t256x2", "r4096_r16x16x16_t128x4"]}
x = torch.randn(1 << 28, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)


def timeit(N):
    batch = (1 << 28) // N
    p = fftc.Plan(N, batch, -1)
    d = p.describe()
    for _ in range(2):
        p.execute(x, y)
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); p.execute(x, y); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    p.close()
    ts.sort()
    return ts[len(ts) // 2], d


for N in [1 << 16, 1 << 20, 1 << 24]:
    for M in sorted(COLS):
        K = N // M
        if N % M or K not in ROWS:
            continue
        os.environ["FFTC_SPLIT_M"] = str(M)
        for c in COLS[M]:
            for r in (ROWS[K] if c == COLS[M][0] else ROWS[K][:1]):
                os.environ["FFTC_COL"], os.environ["FFTC_ROW"] = c, r
                t, d = timeit(N)
                assert c in d and r in d, d
                print(json.dumps({"N": N, "M": M, "K": K, "col": c, "row": r, "us": round(t * 1e6, 1),
                                  "two_pass_frac": round(32 * (1 << 28) / t / 1e9 / 6533.2, 3)}), flush=True)
for k in ("FFTC_SPLIT_M", "FFTC_COL", "FFTC_ROW"):
    os.environ.pop(k, None)
