"""Bounds checks without a sanitizer (compute-sanitizer is not available on this pool): every
kernel family runs on ragged shapes with its output placed between guard regions filled with a
sentinel bit pattern, and its input followed by guard data.  A write past either end of `out`,
or any write to `in`, changes a guard or the input and fails the test; the result must still
match the oracle (an aliasing bug that lands inside `out` fails the parity check instead)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
import paper_2207_06803_b200 as fftc  # noqa: E402

pytestmark = pytest.mark.gpu

GUARD = 4096  # complex elements on each side (32 KB, keeps 16-byte alignment)
SENTINEL = np.float32(-1.2345678e-29)

# (N, batch, env): every kernel family, ragged batches / last tiles
CASES = [
    (64, 77, {}),                                   # warp-shuffle exchange
    (8, 1001, {}), (128, 33, {}), (1024, 9, {}),    # staged / direct compiled schedules
    (2048, 5, {}), (4096, 3, {}),                   # L1::no_allocate loads
    (2187, 3, {}), (3125, 2, {}), (1000, 7, {}),    # odd radices, paired FP32
    (48, 37, {}), (4000, 3, {}),                    # generated single-pass (7-smooth)
    (48, 37, {"FFTC_SMOOTH_JIT": "0"}),             # compiled runtime-schedule kernel
    (143, 37, {}), (1088, 5, {}), (61, 9, {}),      # generated single-pass (primes 11..61)
    (143, 37, {"FFTC_JIT_GENERIC": "1"}),
    (6561, 3, {}), (11 * 4096, 2, {}), (100000, 1, {}),          # generated passes (ragged columns)
    (6561, 3, {"FFTC_JIT_PASS_GENERIC": "1"}),
    (1 << 16, 3, {}), (1 << 22, 1, {}), (1 << 24, 1, {}),       # TMA pass kernels (2^22: register 4096 pass)
    (1 << 24, 1, {"FFTC_PASS_LOGS": "12,12", "FFTC_PASS": "rp4096_r16x16x16_c4"}),  # register pass, later position
    (1 << 20, 1, {"FFTC_PASS_LOGS": "12,8", "FFTC_PASS": "cp4096_q4_r32x32_c8b2"}),  # 4-CTA cluster pass
    (1 << 16, 3, {"FFTC_LARGE": "cluster"}),                     # 8-CTA cluster single pass
    (1 << 16, 5, {"FFTC_LARGE": "cluster", "FFTC_C16_Q": "16"}),  # 16-CTA clusters, two CTAs per SM
]


@pytest.mark.parametrize("N,batch,env", CASES)
def test_no_write_outside_out(N, batch, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    x = synth.uniform_c64(N, batch, seed=N % 1009 + batch)
    n = N * batch
    xin = torch.empty(n + GUARD, dtype=torch.complex64, device="cuda")
    xin[:n].copy_(torch.from_numpy(x.reshape(-1)))
    xin[n:].fill_(complex(3.0, -7.0))
    before = xin.clone()
    out = torch.empty(n + 2 * GUARD, dtype=torch.complex64, device="cuda")
    out.view(torch.float32).fill_(float(SENTINEL))
    for sign in (-1, 1):
        with fftc.Plan(N, batch, sign) as p:
            y = p.execute(xin[:n], out[GUARD:GUARD + n])
        torch.cuda.synchronize()
        g = out.view(torch.float32).cpu().numpy()
        assert np.all(g[:2 * GUARD] == SENTINEL), ("write before out", N, batch, env)
        assert np.all(g[2 * (GUARD + n):] == SENTINEL), ("write past out", N, batch, env)
        assert torch.equal(xin, before), ("input modified", N, batch, env)
        ys = y.cpu().numpy().reshape(batch, N)
        idx = np.unique(np.r_[0, batch - 1, batch // 2])
        err = oracle.rel_l2(ys[idx], oracle.fft_ct(x[idx], sign)).max()
        assert err <= min(oracle.tolerance(N), 2e-6), (N, batch, sign, err, env)
