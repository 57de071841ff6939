"""GPU parity of the distributed six-step (csrc/dist.cu) in loopback mode.

With one GPU, all P virtual ranks run on the current device and the three
all-to-alls become device copies: the pack / column-DFT / twiddle / unpack
kernels and every chunk layout are exercised exactly as with NCCL, against the
fp64 oracle (full O2 up to 2^24, spot bins + Parseval + round trip above).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
import paper_2207_06803_b200 as fftc  # noqa: E402

pytestmark = pytest.mark.gpu


def run_dist(x, sign, P, loopback=True, flags=0):
    N = x.size
    d = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    p = fftc.Plan.dist(N, sign, None, 0, P, loopback=loopback, flags=flags)
    try:
        y = torch.empty_like(d)
        p.execute(d, y)
        torch.cuda.synchronize()
        desc = p.describe()
    finally:
        p.close()
    return y, desc


@pytest.mark.parametrize("N", [1 << 16, 1 << 20, 1 << 22])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("sign", [-1, 1])
def test_six_step_loopback(N, P, sign):
    x = synth.uniform_c64(N, 1, seed=N + P)[0]
    y, desc = run_dist(x, sign, P)
    assert "kind=dist" in desc
    ref = oracle.fft_ct(x[None], sign)[0]
    err = oracle.rel_l2(y.cpu().numpy()[None], ref[None]).max()
    assert err <= oracle.tolerance(N), (N, P, err, desc)
    assert err <= 2e-6


def test_six_step_p1_without_loopback():
    N = 1 << 20
    x = synth.uniform_c64(N, 1, seed=5)[0]
    y, desc = run_dist(x, -1, 1, loopback=False)
    ref = oracle.fft_ct(x[None], -1)[0]
    assert oracle.rel_l2(y.cpu().numpy()[None], ref[None]).max() <= oracle.tolerance(N)


@pytest.mark.parametrize("N,P", [(1 << 24, 8), (1 << 26, 4)])
def test_six_step_large(N, P):
    x = synth.uniform_c64(N, 1, seed=7)[0]
    y, desc = run_dist(x, -1, P)
    yh = y.cpu().numpy()
    if N <= (1 << 24):
        ref = oracle.fft_ct(x[None], -1)[0]
        assert oracle.rel_l2(yh[None], ref[None]).max() <= oracle.tolerance(N)
    else:
        _spot_and_parseval(x, yh, -1)
    # K = K1 K2 path is taken at 2^26
    if N == (1 << 26):
        assert "K2=1 " not in desc


def _spot_and_parseval(x, y, sign, nbins=12):
    N = x.size
    rng = np.random.default_rng(0)
    bins = [0, 1, N // 2, N - 1] + list(rng.integers(0, N, nbins - 4))
    ref = np.array([oracle.spot_bin(x[None], int(k), sign) for k in bins])
    got = y[np.array(bins)].astype(np.complex128)
    # per-bin error relative to the transform's rms magnitude sqrt(N) * rms(x)
    scale = np.sqrt(N) * np.sqrt(np.mean(np.abs(x.astype(np.complex128)) ** 2))
    assert np.abs(got - ref).max() / scale <= oracle.tolerance(N)
    ex = np.sum(np.abs(x.astype(np.complex128)) ** 2)
    ey = np.sum(np.abs(y.astype(np.complex128)) ** 2)
    assert abs(ey - N * ex) / (N * ex) < 1e-5


@pytest.mark.slow
def test_config5_loopback_2p30():
    """BASELINE config 5: N = 2^30 (8 GiB), P = 8 virtual ranks; spot bins, Parseval, round trip."""
    N, P = 1 << 30, 8
    x = synth.uniform_c64(N, 1, seed=0)[0]
    d = torch.from_numpy(x).cuda()
    pf = fftc.Plan.dist(N, -1, None, 0, P, loopback=True)
    y = torch.empty_like(d)
    pf.execute(d, y)
    torch.cuda.synchronize()
    pf.close()
    _spot_and_parseval(x, y.cpu().numpy(), -1, nbins=8)
    pi = fftc.Plan.dist(N, 1, None, 0, P, loopback=True)
    z = torch.empty_like(d)
    pi.execute(y, z)
    torch.cuda.synchronize()
    pi.close()
    del y
    num = torch.linalg.vector_norm(torch.view_as_real(z / N - d).double())
    den = torch.linalg.vector_norm(torch.view_as_real(d).double())
    assert (num / den).item() <= 2 * oracle.tolerance(N)


def transposed_pos(N, P, k):
    """Position of X[k] in the FFTC_DIST_TRANSPOSED_OUT layout:
    out[p*N/P + k1*Mp + jl] = X[p*Mp + jl + M*k1]."""
    M, K, _, _ = fftc.fftc_dist_split(N, P)
    Mp = M // P
    k = np.asarray(k, dtype=np.int64)
    j, k1 = k % M, k // M
    return (j // Mp) * (N // P) + k1 * Mp + j % Mp


@pytest.mark.parametrize("N,P", [(1 << 16, 2), (1 << 20, 4), (1 << 20, 8), (1 << 26, 4)])
@pytest.mark.parametrize("flags", [fftc.FFTC_DIST_PEER_STORES, fftc.FFTC_DIST_TRANSPOSED_OUT,
                                   fftc.FFTC_DIST_PEER_STORES | fftc.FFTC_DIST_TRANSPOSED_OUT])
@pytest.mark.parametrize("sign", [-1, 1])
def test_six_step_fused_exchange_and_transposed_output(N, P, flags, sign):
    """NEXT-1 in loopback: the fused peer-store exchanges (the pack and DFT_M kernels store each
    chunk straight into the receiving rank's buffer) and the transposed output (no
    all-to-all #3), against the oracle; K > 4096 (two-pass DFT_K) at 2^26."""
    x = synth.uniform_c64(N, 1, seed=N + P + flags)[0]
    y, desc = run_dist(x, sign, P, flags=flags)
    assert ("peer-stores" in desc) == bool(flags & fftc.FFTC_DIST_PEER_STORES), desc
    yh = y.cpu().numpy()
    if flags & fftc.FFTC_DIST_TRANSPOSED_OUT:
        assert "output=transposed" in desc and "a2a=2" in desc
        yh = yh[transposed_pos(N, P, np.arange(N))]  # back to natural order
    if N <= (1 << 22):
        ref = oracle.fft_ct(x[None], sign)[0]
        err = oracle.rel_l2(yh[None], ref[None]).max()
        assert err <= min(oracle.tolerance(N), 2e-6), (N, P, flags, err)
    else:
        _spot_and_parseval(x, yh, sign, nbins=8)
