"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle.

Gate (BASELINE.json north_star): per-transform relative L2 <= 2e-6 * log2(N).
Inputs are seeded (synth.py); the oracle sees exactly the fp32 array the GPU gets.
"""
import math

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
import paper_2207_06803_b200 as fftc  # noqa: E402

pytestmark = pytest.mark.gpu


def gpu_fft(x, sign, N=None):
    """x: numpy complex64 (batch, N) -> numpy complex64 via fftc (device buffers)."""
    batch, n = x.shape
    d = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    with fftc.Plan(n, batch, sign) as p:
        y = p(d)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def check(y, x, sign, idx=None, ref="ct"):
    N = x.shape[1]
    xs = x if idx is None else x[idx]
    yr = oracle.fft_ct(xs, sign) if ref == "ct" else oracle.dft_naive(xs, sign)
    ys = y if idx is None else y[idx]
    err = oracle.rel_l2(ys, yr)
    tol = oracle.tolerance(N)
    assert err.max() <= tol, (N, sign, float(err.max()), tol)
    # an fp32 FFT sits near 1e-7; 10x that is a bug even when it passes the gate
    assert err.max() <= 2e-6, (N, sign, float(err.max()))
    return float(err.max())


def sample_idx(batch, seed=0, n_rand=48):
    rng = np.random.default_rng(seed)
    idx = set(range(min(8, batch))) | set(range(max(0, batch - 8), batch))
    if batch > 16:
        idx |= set(rng.integers(0, batch, n_rand).tolist())
    return np.array(sorted(idx), dtype=np.int64)


POW2 = [1 << k for k in range(3, 13)]
MIXED = [60, 105, 210, 1000, 2187, 3125]
GENERIC = [2, 3, 4, 5, 6, 7, 12, 24, 27, 35, 48, 49, 81, 100, 125, 243, 343, 360, 500, 729, 1344, 2401,
           3000, 3072, 4000]


# ---------------------------------------------------------------- config 1
def test_config1_full():
    """BASELINE config 1: N=64, batch=4096, U[-1,1) seed 0, forward; every transform."""
    x = synth.uniform_c64(64, 4096, seed=0)
    y = gpu_fft(x, -1)
    check(y, x, -1)


# ---------------------------------------------------------------- small batches incl. ragged tails
@pytest.mark.parametrize("N", POW2 + MIXED + GENERIC)
@pytest.mark.parametrize("batch", [1, 3, 7, 64])
@pytest.mark.parametrize("sign", [-1, 1])
def test_small_batches(N, batch, sign):
    x = synth.uniform_c64(N, batch, seed=N * 131 + batch)
    y = gpu_fft(x, sign)
    check(y, x, sign)


@pytest.mark.parametrize("N", [1 << 16, 1 << 20])
@pytest.mark.parametrize("sign", [-1, 1])
@pytest.mark.parametrize("large", ["l2", "passes", "fourstep"])
def test_fourstep_small_batch(N, sign, large, monkeypatch):
    monkeypatch.setenv("FFTC_LARGE", large)
    x = synth.normal_c64(N, 3, seed=N)
    with fftc.Plan(N, 3, sign) as p:
        assert ("kind=" + large) in p.describe()
    y = gpu_fft(x, sign)
    check(y, x, sign)


@pytest.mark.parametrize("n", list(range(13, 25)))
def test_multipass_all_pow2(n):
    """Every power of two 2^13..2^24 on the default large-N path (HBM multi-pass), both
    signs, odd batch."""
    N = 1 << n
    batch = max(1, (1 << 22) // N) | 1
    x = synth.uniform_c64(N, batch, seed=n)
    for sign in (-1, 1):
        y = gpu_fft(x, sign)
        idx = sample_idx(batch, n_rand=4)
        check(y[idx], x[idx], sign)


@pytest.mark.parametrize("n,name", [(17, "p512_r32x16_c8"), (18, "p512_r32x16_c8"), (18, "p512_r16x32_c8t32"),
                                    (19, "p1024_r32x32_c8b1"), (20, "p1024_r32x32_c8b1"),
                                    (20, "p1024_r32x32_c8b2")])
def test_every_pass_candidate(n, name, monkeypatch):
    """Each compiled 8-column pass kernel (L = 512 / 1024, TMA boxes split at 256 rows)."""
    monkeypatch.setenv("FFTC_PASS", name)
    N = 1 << n
    batch = 3
    x = synth.uniform_c64(N, batch, seed=n)
    with fftc.Plan(N, batch, -1) as p:
        assert name in p.describe(), p.describe()
    for sign in (-1, 1):
        check(gpu_fft(x, sign), x, sign)


@pytest.mark.parametrize("n,name", [(16, "p256_r16x16_b3m2"), (24, "p256_r16x16_b3m2"), (14, "p128_r16x8_b3m4"),
                                    (14, "p128_r16x8_b4m3"), (18, "p512_r16x32_c8t32b3"),
                                    (20, "p1024_r32x32_c8b3"), (16, "p256_r16x16_b2m2"), (20, "p1024_r32x32_c8b2")])
def test_pass_buffer_ring_wraps(n, name, monkeypatch):
    """Pass kernels with 2-4 tile buffers on 2^24 elements: every persistent CTA runs many
    tiles, so each buffer is refilled (and its mbarrier phase flips) several times; sampled
    transforms against the oracle, both signs."""
    monkeypatch.setenv("FFTC_PASS", name)
    N = 1 << n
    batch = (1 << 24) // N
    x = synth.uniform_c64(N, batch, seed=n + 7)
    with fftc.Plan(N, batch, -1) as p:
        assert name in p.describe(), p.describe()
    idx = sample_idx(batch, n_rand=3)
    for sign in (-1, 1):
        check(gpu_fft(x, sign)[idx], x[idx], sign)


@pytest.mark.parametrize("logs,later", [("12,12", None), ("11,11", None), ("11,11", "p2048_r16x16x8_c2b3"),
                                        ("12,11", None), ("11,10", None), ("10,11", None), ("12,8", None),
                                        ("8,12", None), ("12,6,6", None), ("11,9,4", None), ("8,11,4", None),
                                        ("12,12", "p4096_r16x16x16_c4b1")])
def test_long_pass_narrow_tiles(logs, later, monkeypatch):
    """2048/4096-long passes (2/4-column tiles, 16/32-byte TMA rows, swizzled exchanges): forced
    splits of 2^16..2^24, first and later positions, sampled transforms vs the oracle."""
    monkeypatch.setenv("FFTC_PASS_LOGS", logs)
    if later:
        monkeypatch.setenv("FFTC_PASS", later)
    n = sum(int(e) for e in logs.split(","))
    N = 1 << n
    batch = max(1, (1 << 23) // N) | 1
    x = synth.uniform_c64(N, batch, seed=n + 11)
    with fftc.Plan(N, batch, -1) as p:
        d = p.describe()
        for e in logs.split(","):
            assert "p%d_" % (1 << int(e)) in d, d
    idx = sample_idx(batch, n_rand=3)
    for sign in (-1, 1):
        check(gpu_fft(x, sign)[idx], x[idx], sign)


@pytest.mark.parametrize("logs,batch", [("12,8", 17), ("8,12", 17), ("12,10", 5), ("12,12", 1)])
def test_cluster_pass(logs, batch, monkeypatch):
    """The 4096-long pass on a cluster of four CTAs (cpass.cu: rows = q mod 4 per CTA, 1024-point
    sub-DFTs, peer-shared bulk-copy exchange, radix-4 combine), first and later positions; the
    persistent clusters run several tiles each (mbarrier phases flip), sampled vs the oracle."""
    monkeypatch.setenv("FFTC_PASS_LOGS", logs)
    monkeypatch.setenv("FFTC_PASS", "cp4096_q4_r32x32_c8b2")
    n = sum(int(e) for e in logs.split(","))
    N = 1 << n
    x = synth.uniform_c64(N, batch, seed=n + 13)
    with fftc.Plan(N, batch, -1) as p:
        assert "cp4096_q4_r32x32_c8b2" in p.describe(), p.describe()
    idx = sample_idx(batch, n_rand=3)
    for sign in (-1, 1):
        check(gpu_fft(x, sign)[idx], x[idx], sign)


@pytest.mark.parametrize("logs,batch", [("12,8", 17), ("8,12", 17), ("12,10", 5), ("11,12", 3), ("12,12", 1),
                                        ("12,12", 2), ("12,4", 1), ("4,12", 3)])
def test_register_pass(logs, batch, monkeypatch):
    """The 4096-long pass with its tile held in registers (rpass.cu: 4-column tiles, two-half
    stage exchanges, outputs stored from registers), first and later positions, persistent CTAs
    running many tiles (the mbarrier phase flips), sampled vs the oracle, both signs."""
    monkeypatch.setenv("FFTC_PASS_LOGS", logs)
    name = "rp4096_r16x16x16_c4"
    monkeypatch.setenv("FFTC_PASS", name)
    n = sum(int(e) for e in logs.split(","))
    N = 1 << n
    x = synth.uniform_c64(N, batch, seed=n + 17)
    with fftc.Plan(N, batch, -1) as p:
        assert name + " " in p.describe() or name + "," in p.describe(), p.describe()
    idx = sample_idx(batch, n_rand=3)
    for sign in (-1, 1):
        check(gpu_fft(x, sign)[idx], x[idx], sign)


@pytest.mark.parametrize("q", ["8", "16"])
@pytest.mark.parametrize("batch", [1, 3, 17, 40])
def test_cluster_single_pass_65536(batch, q, monkeypatch):
    """N = 65536 in one HBM round trip on a cluster of eight CTAs (c16.cu: column DFT_256 per CTA,
    rows delivered to their owner CTA through distributed shared memory, row DFT_256 with the
    folded w_N^{rj}); batches above the number of resident clusters make every cluster run
    several transforms (mbarrier phases and cluster-barrier rounds wrap), both signs; clusters of 8
    (one CTA per SM) and of 16 (two CTAs per SM)."""
    monkeypatch.setenv("FFTC_LARGE", "cluster")
    monkeypatch.setenv("FFTC_C16_Q", q)
    N = 1 << 16
    x = synth.normal_c64(N, batch, seed=batch + 29)
    with fftc.Plan(N, batch, -1) as p:
        assert "kind=cluster" in p.describe(), p.describe()
    idx = sample_idx(batch, n_rand=4)
    for sign in (-1, 1):
        check(gpu_fft(x, sign)[idx], x[idx], sign)


# ---------------------------------------------------------------- the paper's own check
def test_paper_protocol_p217_on_gpu():
    """The paper's accuracy experiment on the GPU path: random inputs, N = 32..1024,
    ten runs each, max |result - reference| / N < 1e-7 -- with the fp64 oracle as the
    reference (the paper compared against numpy) and the fp32 GPU result."""
    for N in [32, 64, 128, 256, 512, 1024]:
        x = synth.uniform_c64(N, 10, seed=1000 * N)
        for sign in (-1,):
            y = gpu_fft(x, sign).astype(np.complex128)
            ref = oracle.fft_ct(x, sign)
            assert (np.abs(y - ref).max(axis=1) / N < 1e-7).all(), N


# ---------------------------------------------------------------- random large sizes
def _random_large_sizes(count=24, seed=2207):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        e = rng.integers(0, [23, 12, 8, 6])  # 2^a 3^b 5^c 7^d
        n = 2 ** int(e[0]) * 3 ** int(e[1]) * 5 ** int(e[2]) * 7 ** int(e[3])
        if 4096 < n <= (1 << 22):
            out.append(n)
    return sorted(set(out))


@pytest.mark.parametrize("N", _random_large_sizes())
def test_random_large_sizes(N):
    """Seeded random 7-smooth N in (4096, 2^22]: whichever large-N path the planner picks
    (TMA passes or runtime passes), ragged batch, both signs, against the oracle."""
    batch = max(1, (1 << 21) // N) | 1
    x = synth.uniform_c64(N, batch, seed=N % 1009)
    idx = np.array(sorted({0, batch // 2, batch - 1}))
    for sign in (-1, 1):
        y = gpu_fft(x, sign)
        check(y[idx], x[idx], sign)


# ---------------------------------------------------------------- beyond 2^31 elements
@pytest.mark.parametrize("N,batch", [(64, (1 << 25) + 3), (4096, (1 << 19) + 5), (1 << 16, (1 << 15) + 1)])
def test_more_than_2p31_elements(N, batch):
    """batch*N > 2^31 (16 GiB buffers): 64-bit offsets in every kernel / tensor map.  Input
    drawn on the device from a seeded generator; the oracle checks transforms sampled across
    the whole batch, the last ones included."""
    g = torch.Generator(device="cuda").manual_seed(N)
    d = (torch.rand(batch * N * 2, device="cuda", generator=g, dtype=torch.float32) * 2 - 1).view(torch.complex64)
    with fftc.Plan(N, batch, -1) as p:
        y = p(d)
    torch.cuda.synchronize()
    idx = np.array([0, 1, batch // 3, batch // 2, (1 << 31) // N - 1, (1 << 31) // N, batch - 2, batch - 1])
    xs = d.view(batch, N)[torch.from_numpy(idx).cuda()].cpu().numpy()
    ys = y.view(batch, N)[torch.from_numpy(idx).cuda()].cpu().numpy()
    del d, y
    torch.cuda.empty_cache()
    check(ys, xs, -1)


# ---------------------------------------------------------------- every single-pass size
def _smooth7(n):
    for q in (2, 3, 5, 7):
        while n % q == 0:
            n //= q
    return n == 1


ALL_SMOOTH = [n for n in range(2, 4097) if _smooth7(n)]


def test_every_7smooth_size_up_to_4096():
    """Every 7-smooth N <= 4096 the planner accepts (247 sizes; compiled or runtime
    schedule), batch 3, both signs, against the oracle."""
    worst = 0.0
    for N in ALL_SMOOTH:
        x = synth.uniform_c64(N, 3, seed=N)
        for sign in (-1, 1):
            y = gpu_fft(x, sign)
            worst = max(worst, check(y, x, sign))
    assert worst <= 2e-6


# ---------------------------------------------------------------- any 7-smooth N > 4096
GPASS = [(12288, 9), (13122, 7), (15625, 5), (16807, 5), (19683, 5), (40960, 3), (46656, 3), (59049, 3),
         (78125, 2), (100000, 2), (248832, 2), (10 ** 6, 1), (3 ** 13, 1)]


@pytest.mark.parametrize("N,batch", GPASS)
def test_gpass_non_pow2_large(N, batch):
    """Non-power-of-two N above the single-pass limit: runtime-schedule passes (gpass.cu),
    odd row pitches, ragged column tiles, both signs, against the oracle."""
    x = synth.uniform_c64(N, batch, seed=N % 1000)
    with fftc.Plan(N, batch, -1) as p:
        assert "kind=gpass" in p.describe(), p.describe()
        assert p.launches() == len(fftc.fftc_plan_gpasses(N))
    for sign in (-1, 1):
        check(gpu_fft(x, sign), x, sign)


@pytest.mark.parametrize("n", [13, 16, 20])
def test_gpass_forced_pow2(n, monkeypatch):
    """The runtime-schedule passes on powers of two (FFTC_LARGE=gpass) against the oracle."""
    monkeypatch.setenv("FFTC_LARGE", "gpass")
    N = 1 << n
    x = synth.uniform_c64(N, 3, seed=n)
    with fftc.Plan(N, 3, 1) as p:
        assert "kind=gpass" in p.describe()
    check(gpu_fft(x, 1), x, 1)


def test_gpass_config4_sized():
    """A C4-sized non-power-of-two transform: 3^15 (two 243-passes would not fit: three passes)."""
    N = 3 ** 15
    x = synth.normal_c64(N, 1, seed=15)
    with fftc.Plan(N, 1, -1) as p:
        assert "kind=gpass" in p.describe()
    y = gpu_fft(x, -1)
    check(y, x, -1)


# ---------------------------------------------------------------- L2-resident multi-pass path
L2_CASES = [(13, 83), (14, 37), (15, 21), (16, 11), (17, 7), (18, 5), (19, 4), (20, 3), (21, 2)]


@pytest.mark.parametrize("n,batch", L2_CASES)
def test_l2_path_many_chunks(n, batch, monkeypatch):
    """L2-resident path with 1 MiB chunks: many chunks, ragged last chunk, the ring of
    workspace slots wraps several times; both signs against the oracle."""
    monkeypatch.setenv("FFTC_L2_CHUNK_MB", "1")
    monkeypatch.setenv("FFTC_LARGE", "l2")
    N = 1 << n
    x = synth.uniform_c64(N, batch, seed=100 + n)
    with fftc.Plan(N, batch, -1) as p:
        assert "kind=l2" in p.describe(), p.describe()
    idx = np.array(sorted({0, 1, batch // 2, batch - 2, batch - 1}), dtype=np.int64)
    for sign in (-1, 1):
        y = gpu_fft(x, sign)
        check(y[idx], x[idx], sign)


@pytest.mark.parametrize("n", [13, 16, 17, 20])
def test_l2_matches_hbm_multipass(n, monkeypatch):
    """The L2-resident kernel runs the same pass tiles (passtile.cuh, same radices and
    twiddle tables) as the HBM multi-pass kernels: the two agree to fp32 rounding
    (not bitwise: the compiler may contract differently inside the two kernels)."""
    N = 1 << n
    batch = max(2, (1 << 22) // N) + 1
    x = synth.uniform_c64(N, batch, seed=n)
    monkeypatch.setenv("FFTC_L2_CHUNK_MB", "2")
    monkeypatch.setenv("FFTC_LARGE", "l2")
    y_l2 = gpu_fft(x, -1)
    monkeypatch.setenv("FFTC_LARGE", "passes")
    monkeypatch.setenv("FFTC_PASS_MAXLOG", "8")  # the same pass lengths as the L2 split
    y_hbm = gpu_fft(x, -1)
    d = oracle.rel_l2(y_l2, y_hbm.astype(np.complex128))
    assert d.max() <= 2e-7, float(d.max())


@pytest.mark.parametrize("n", [25, 26, 27, 28])
def test_multipass_three_long_passes(n):
    """2^25..2^28: three passes, 512/1024-long (8-column) tiles then a 256-long (16-column)
    last pass.  Spot bins by direct summation (the definition), Parseval, and the round trip."""
    N = 1 << n
    x = synth.uniform_c64(N, 1, seed=n)
    with fftc.Plan(N, 1, -1) as p:
        assert "kind=passes" in p.describe() and p.launches() == 3, p.describe()
    d = torch.from_numpy(x).cuda()
    with fftc.Plan(N, 1, -1) as pf, fftc.Plan(N, 1, 1) as pi:
        y = pf(d)
        z = pi(y)
    torch.cuda.synchronize()
    yh = y.cpu().numpy()[0]
    rng = np.random.default_rng(n)
    scale = np.sqrt(N) * np.sqrt(np.mean(np.abs(x.astype(np.complex128)) ** 2))
    for k in [0, 1, N // 2, N - 1] + rng.integers(0, N, 6).tolist():
        ref = oracle.spot_bin(x, int(k), -1)
        assert abs(yh[k] - ref) / scale <= 2e-6, (n, k)
    ex = np.sum(np.abs(x.astype(np.complex128)) ** 2)
    ey = np.sum(np.abs(yh.astype(np.complex128)) ** 2)
    assert abs(ey / (N * ex) - 1) < 1e-5
    rt = z.cpu().numpy()[0].astype(np.complex128) / N
    err = np.sqrt(np.sum(np.abs(rt - x[0]) ** 2) / ex)
    assert err <= 2 * oracle.tolerance(N), err


@pytest.mark.parametrize("N", POW2 + MIXED)
def test_every_candidate_schedule(N, monkeypatch):
    """Every compiled schedule (not just the planner's default) is correct, both signs, ragged batch."""
    names = fftc.fftc_candidates(N)
    assert names
    x = synth.uniform_c64(N, 37, seed=N)
    for name in names:
        monkeypatch.setenv("FFTC_KERNEL", name)
        for sign in (-1, 1):
            with fftc.Plan(N, 37, sign) as p:
                assert name in p.describe()
                y = p(torch.from_numpy(x).cuda())
            torch.cuda.synchronize()
            check(y.cpu().numpy(), x, sign)


# ---------------------------------------------------------------- full BASELINE sizes (sampled)
@pytest.mark.parametrize("N", POW2)
@pytest.mark.parametrize("sign", [-1, 1])
def test_config2_full_size(N, sign):
    """BASELINE config 2: batch = 2^26/N; sampled transforms vs O2, plus a whole-buffer Parseval check."""
    batch = (1 << 26) // N
    x = synth.uniform_c64(N, batch, seed=0)
    d = torch.from_numpy(x).cuda()
    with fftc.Plan(N, batch, sign) as p:
        yd = p(d)
    torch.cuda.synchronize()
    # Parseval over every transform (torch reductions on device: checking, not computing)
    ex = (d.abs() ** 2).double().sum(dim=1)
    ey = (yd.abs() ** 2).double().sum(dim=1)
    rel = ((ey - N * ex).abs() / (N * ex)).max().item()
    assert rel < 1e-5
    idx = sample_idx(batch)
    y = yd[torch.from_numpy(idx).cuda()].cpu().numpy()
    check(np.asarray(y), x[idx], sign)


@pytest.mark.parametrize("N", MIXED)
def test_config3_full_size(N):
    batch = (1 << 26) // N
    x = synth.uniform_c64(N, batch, seed=0)
    d = torch.from_numpy(x).cuda()
    with fftc.Plan(N, batch, -1) as p:
        yd = p(d)
    torch.cuda.synchronize()
    idx = sample_idx(batch)
    y = yd[torch.from_numpy(idx).cuda()].cpu().numpy()
    check(y, x[idx], -1)


@pytest.mark.parametrize("N", [1 << 16, 1 << 20, 1 << 24])
def test_config4_round_trip(N):
    """BASELINE config 4: batch = 2^28/N, N(0,1) values; forward then inverse round trip."""
    batch = (1 << 28) // N
    x = synth.normal_c64(N, batch, seed=0)
    d = torch.from_numpy(x).cuda()
    del x
    with fftc.Plan(N, batch, -1) as pf, fftc.Plan(N, batch, 1) as pi:
        yd = pf(d)
        zd = pi(yd)
    torch.cuda.synchronize()
    tol = oracle.tolerance(N)
    # sampled forward transforms vs O2
    ns = {1 << 16: 6, 1 << 20: 3, 1 << 24: 1}[N]
    idx = np.unique(np.array([0, batch - 1] + list(np.random.default_rng(1).integers(0, batch, ns))))
    xi = d[torch.from_numpy(idx).cuda()].cpu().numpy()
    yi = yd[torch.from_numpy(idx).cuda()].cpu().numpy()
    check(yi, xi, -1)
    # inverse applied to the GPU forward output, vs O2(y_gpu, +1)
    zi = zd[torch.from_numpy(idx).cuda()].cpu().numpy()
    zr = oracle.fft_ct(yi, +1)
    assert oracle.rel_l2(zi, zr).max() <= tol
    # whole-buffer round trip inv(fwd(x))/N = x
    num = ((zd / N - d).abs() ** 2).double().sum(dim=1).sqrt()
    den = (d.abs() ** 2).double().sum(dim=1).sqrt()
    assert (num / den).max().item() <= 2 * tol


# ---------------------------------------------------------------- special inputs
@pytest.mark.parametrize("N", [8, 64, 60, 105, 1000, 3125, 4096, 1 << 16])
def test_special_inputs(N):
    batch = 4
    d = np.zeros((batch, N), np.complex64)
    d[:, 0] = 1
    y = gpu_fft(d, -1)
    assert np.array_equal(y, np.ones_like(y))  # delta -> exactly ones
    z = gpu_fft(np.zeros((batch, N), np.complex64), -1)
    assert np.array_equal(z, np.zeros_like(z))  # zero -> exactly zero
    k0 = (3 * N) // 7
    n = np.arange(N)
    tone = np.exp(2j * np.pi * ((k0 * n) % N) / N).astype(np.complex64)
    t = gpu_fft(np.tile(tone, (batch, 1)), -1)
    ref = np.zeros(N); ref[k0] = N
    assert (np.linalg.norm(t - ref, axis=1) / N).max() <= oracle.tolerance(N)
    # linearity
    a = synth.uniform_c64(N, batch, seed=1)
    b = synth.uniform_c64(N, batch, seed=2)
    ya, yb = gpu_fft(a, -1), gpu_fft(b, -1)
    yab = gpu_fft((a + b).astype(np.complex64), -1)
    assert oracle.rel_l2(yab, ya.astype(np.complex128) + yb).max() <= oracle.tolerance(N)


def test_n1_and_batch0():
    x = synth.uniform_c64(1, 5, seed=0)
    assert np.array_equal(gpu_fft(x, -1), x)
    with fftc.Plan(64, 0, -1) as p:
        t = torch.zeros(16, dtype=torch.complex64, device="cuda")
        assert fftc.fftc_execute(p.handle, t.data_ptr(), t[8:].data_ptr(), 0) == fftc.FFTC_SUCCESS


def test_boundary_errors():
    N, batch = 64, 16
    x = torch.zeros(N * batch + 8, dtype=torch.complex64, device="cuda")
    y = torch.zeros(N * batch + 8, dtype=torch.complex64, device="cuda")
    with fftc.Plan(N, batch, -1) as p:
        h = p.handle
        assert fftc.fftc_execute(h, 0, y.data_ptr(), 0) == fftc.FFTC_ERROR_INVALID_VALUE
        assert fftc.fftc_execute(h, x.data_ptr(), x.data_ptr(), 0) == fftc.FFTC_ERROR_INVALID_VALUE
        assert fftc.fftc_execute(h, x.data_ptr(), x.data_ptr() + 8 * 8, 0) == fftc.FFTC_ERROR_INVALID_VALUE
        assert fftc.fftc_execute(h, x.data_ptr() + 8, y.data_ptr(), 0) == fftc.FFTC_ERROR_MISALIGNED
        assert fftc.fftc_execute(h, x.data_ptr(), y.data_ptr() + 8, 0) == fftc.FFTC_ERROR_MISALIGNED
        assert fftc.fftc_execute(h, x.data_ptr(), y.data_ptr(), 0) == fftc.FFTC_SUCCESS
    for bad, code in [((0, 1, -1), 1), ((8, 1, 0), 1), ((67, 1, -1), 2), ((8 * 67, 1, -1), 2)]:
        assert fftc.fftc_plan_create(*bad) == 0
        assert fftc.fftc_last_error() == code
    torch.cuda.synchronize()


def test_describe_and_launches():
    for N, kind, launches in [(64, "fused", 1), (4096, "fused", 1), (48, "jit", 1), (1 << 20, "passes", 2),
                              (1 << 24, "passes", 3), (1 << 13, "passes", 2), (1 << 16, "passes", 2),
                              (1 << 22, "passes", 2), (1 << 23, "passes", 2)]:
        with fftc.Plan(N, 2, -1) as p:
            assert ("kind=" + kind) in p.describe()
            assert p.launches() == launches


def test_execute_host_matches_device():
    N, batch = 1000, 2000
    x = synth.uniform_c64(N, batch, seed=3)
    out = np.empty_like(x)
    with fftc.Plan(N, batch, -1) as p:
        p.execute_host(x, out)
    y = gpu_fft(x, -1)
    assert np.array_equal(out, y)  # same kernels, same result bit for bit
    idx = sample_idx(batch)
    check(out[idx], x[idx], -1)


def test_execute_host_matches_device_l2(monkeypatch):
    """Host-staged execution of an L2-path plan (each staging slot owns its ring + counters)."""
    monkeypatch.setenv("FFTC_LARGE", "l2")
    N, batch = 1 << 16, 150
    x = synth.uniform_c64(N, batch, seed=4)
    out = np.empty_like(x)
    with fftc.Plan(N, batch, 1) as p:
        assert "kind=l2" in p.describe()
        p.execute_host(x, out)
    y = gpu_fft(x, 1)
    assert np.array_equal(out, y)
    idx = np.array([0, 63, 64, 149])
    check(out[idx], x[idx], 1)


def test_determinism_bitwise():
    x = synth.uniform_c64(4096, 256, seed=9)
    a = gpu_fft(x, -1)
    b = gpu_fft(x, -1)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- negative controls of the gate
@pytest.mark.parametrize("N", [64, 3125, 4096, 1 << 16])
def test_check_rejects_wrong_gpu_output(N):
    """check() (the parity gate every test and smoke() use) passes the real fftc output and
    raises on wrong ones derived from it: one bin perturbed by 10*tol*||y||, the conjugated
    spectrum, two bins swapped, and the output of the opposite sign (the error
    check the gate descends from)."""
    batch = 6
    x = synth.uniform_c64(N, batch, seed=11)
    y = gpu_fft(x, -1)
    check(y, x, -1)  # positive control
    tol = oracle.tolerance(N)
    bad = y.copy()
    bad[3, N // 3] += np.complex64(10 * tol * np.linalg.norm(y[3]))
    wrong = [bad, np.conj(y)]
    sw = y.copy()
    sw[:, [1, N - 1]] = sw[:, [N - 1, 1]]
    wrong.append(sw)
    wrong.append(gpu_fft(x, +1))
    for w in wrong:
        with pytest.raises(AssertionError):
            check(w, x, -1)


def test_binding_rejects_short_and_wrong_tensors():
    """The binding checks sizes, dtype, contiguity and device before handing bare pointers to
    the C ABI (a short buffer would otherwise be read or written past its end)."""
    N, batch = 256, 8
    with fftc.Plan(N, batch, -1) as p:
        x = torch.zeros(N * batch, dtype=torch.complex64, device="cuda")
        with pytest.raises(ValueError):
            p(x[: N * batch - 1])
        with pytest.raises(ValueError):
            p.execute(x, torch.empty(N * batch - 1, dtype=torch.complex64, device="cuda"))
        with pytest.raises(TypeError):
            p.execute(x, torch.empty(2 * N * batch, dtype=torch.float32, device="cuda"))
        with pytest.raises(TypeError):
            p.execute(x, torch.empty(2 * N * batch, dtype=torch.complex64, device="cuda")[::2])
        with pytest.raises(TypeError):
            p.execute(x.cpu(), torch.empty_like(x))
        with pytest.raises(ValueError):
            p.execute_host(np.zeros(N * batch - 1, np.complex64), np.zeros(N * batch, np.complex64))
        with pytest.raises(TypeError):
            p.execute_host(x, np.zeros(N * batch, np.complex64))
        y = p(x)  # the well-formed call still works
        assert y.numel() == N * batch


def test_execute_host_many_chunks(monkeypatch):
    """fftc_execute_host with 1 MiB chunks over a 128 MiB host buffer (> 64 chunks: the chunk-size
    ramp must stay capped) equals the device execution bit for bit."""
    monkeypatch.setenv("FFTC_HOST_CHUNK_MB", "1")
    N, batch = 4096, 4096  # 128 MiB
    x = synth.uniform_c64(N, batch, seed=12)
    out = np.empty_like(x)
    with fftc.Plan(N, batch, -1) as p:
        p.execute_host(x, out)
    assert np.array_equal(out, gpu_fft(x, -1))
    idx = sample_idx(batch)
    check(out[idx], x[idx], -1)


@pytest.mark.parametrize("N", [48, 360, 2401, 4000])
def test_compiled_runtime_schedule_kernel(N, monkeypatch):
    """FFTC_SMOOTH_JIT=0: 7-smooth N without a compiled schedule on the compiled runtime-schedule
    kernel (k_generic, the path when NVRTC is missing), ragged batch, both signs."""
    monkeypatch.setenv("FFTC_SMOOTH_JIT", "0")
    x = synth.uniform_c64(N, 7, seed=N)
    for sign in (-1, 1):
        with fftc.Plan(N, 7, sign) as p:
            assert "kind=generic" in p.describe(), p.describe()
            y = p(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        check(y.cpu().numpy(), x, sign)
