"""CPU pins of the index algebra of the round-2 large-N kernels (no GPU).

rpass.cu (the 4096-long pass with its tile in registers) and c16.cu (N = 65536 on a cluster) rely
on facts that are easy to get wrong and hard to see in a failing GPU run: which half of the stage
exchange each butterfly writes, that the swizzled exchange layout is a bijection without bank
conflicts, that folding an input twiddle into the Stockham stages' twiddles is an identity, and that
the cluster's row delivery covers every element once.  Each is checked here in numpy, in float64,
against numpy's FFT where a transform is involved (Eq. 2; DESIGN §6 K2 / K6).
"""
import numpy as np
import pytest

L, R, NB, HALF = 4096, 16, 256, 2048


def st_pos(j, r, Ns):
    """Stockham write position of output r of butterfly j (stage with Ns, L' = 16 Ns)."""
    return (j // Ns) * (R * Ns) + (j % Ns) + r * Ns


def ex_idx(p, f, C=4):
    p = p % HALF
    return (((p & (HALF - 16)) | ((p & 15) ^ ((p >> 4) & 15)))) * C + f


@pytest.mark.parametrize("Ns", [1, 16])
def test_rpass_exchange_halves(Ns):
    """Thread (f, jl) owns butterflies jl and jl + 128: the first writes only p < 2048, the second
    only p >= 2048, every position is written once, and the readers' slots r' < 8 are p < 2048."""
    r = np.arange(R)
    seen = np.zeros(L, int)
    for jl in range(128):
        a = st_pos(jl, r, Ns)
        b = st_pos(jl + 128, r, Ns)
        assert (a < HALF).all() and (b >= HALF).all(), (jl, Ns)
        seen[a] += 1
        seen[b] += 1
    assert (seen == 1).all()
    for jl in range(128):
        for k in (0, 1):
            pos = jl + 128 * k + NB * r
            assert (pos[:8] < HALF).all() and (pos[8:] >= HALF).all()


def _half_warp_slots(addrs):
    """8-byte accesses of 16 lanes: distinct 8-byte bank slots (mod 16) means no conflict."""
    return len(set(int(a) % 16 for a in addrs)) == len(addrs)


def test_rpass_exchange_layout_bijective_and_conflict_free():
    idx = {ex_idx(p, f) for p in range(HALF) for f in range(4)}
    assert idx == set(range(HALF * 4))
    # lanes of a half-warp: f = lane % 4, jl = base + lane // 4 (4 consecutive butterflies)
    for base in range(0, 128, 4):
        lanes = [(l % 4, base + l // 4) for l in range(16)]
        for Ns in (1, 16):
            for r in range(R):  # stage writes (half A: butterfly jl)
                assert _half_warp_slots([ex_idx(st_pos(j, r, Ns), f) for f, j in lanes]), (base, Ns, r)
        for k in (0, 1):
            for rr in range(8):  # stage reads x[j + 128 k + 256 r']
                assert _half_warp_slots([ex_idx(j + 128 * k + NB * rr, f) for f, j in lanes])


def _stockham(x, radices, tw_in):
    """Stockham DFT along axis -1 with radices (R_0 first); tw_in(s, j, r) -> extra input factor
    of stage s, butterfly j, input r (1 for a plain DFT); stage twiddle w_{L'}^{(j mod Ns) r}."""
    n = x.shape[-1]
    a = x.astype(np.complex128)
    Ns = 1
    for s, Rs in enumerate(radices):
        nb = n // Rs
        j = np.arange(nb)[:, None]
        r = np.arange(Rs)[None, :]
        v = a[..., j + r * nb]  # (..., nb, Rs)
        Lp = Ns * Rs
        v = v * np.exp(-2j * np.pi * ((j % Ns) * r) / Lp) * tw_in(s, j, r)
        y = np.fft.fft(v, axis=-1)
        b = np.empty_like(a)
        b[..., (j // Ns) * Lp + (j % Ns) + r * Ns] = y
        a = b
        Ns = Lp
    return a


@pytest.mark.parametrize("Ns_pass,m", [(4096, 1), (4096, 2731), (512, 77), (1 << 20, 654321)])
def test_rpass_folded_input_twiddle(Ns_pass, m):
    """rpass later pass: DFT_4096 of x[i] w_T^{m i} (T = Ns L) equals the three radix-16 stages
    with stage s's input r multiplied by u_s^r: u_0 = w_T^{256 m}, u_1 = w_T^{16 m} w_256^{j1 mod 16}
    (the stage-1 twiddle absorbed), u_2 = w_T^{m} w_4096^{j2} (likewise)."""
    T = Ns_pass * L
    rng = np.random.default_rng(m)
    x = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    w = lambda e: np.exp(-2j * np.pi * (np.asarray(e) % T) / T)
    ref = np.fft.fft(x * w(m * np.arange(L)))

    def tw_in(s, j, r):
        if s == 0:
            return w(NB * m * r)
        if s == 1:  # the stage twiddle w_256^{(j mod 16) r} is applied by _stockham; the fold adds w_T^{16 m r}
            return w(16 * m * r)
        return w(m * r)  # stage 2: w_4096^{j r} by _stockham, the fold adds w_T^{m r}

    got = _stockham(x, [16, 16, 16], tw_in)
    assert np.abs(got - ref).max() < 1e-9 * np.abs(ref).max()


def test_c16_folded_row_twiddle():
    """c16: the four-step 256 x 256 with w_N^{r j} folded into the row DFT (stage B1 input s times
    w_N^{16 j s}, stage B2 input s2 times w_N^{(256 i2 + j) s2} in place of w_256^{i2 s2}) equals
    the DFT of N = 65536."""
    N, S = 65536, 256
    rng = np.random.default_rng(2207)
    x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    A = x.reshape(S, S)  # A[q][r] = x[256 q + r]
    Y = np.fft.fft(A, axis=0)  # Y[j][r]: DFT_256 down each column r
    wN = lambda e: np.exp(-2j * np.pi * (np.asarray(e) % N) / N)
    j = np.arange(S)[:, None]
    # row DFT over r of Y[j][r] w_N^{r j}: two radix-16 stages with the folded factors
    out = np.empty((S, S), complex)
    for jj in range(S):
        def tw_in(s, i, rr, jj=jj):
            if s == 0:
                return wN(16 * jj * rr)
            # _stockham applies w_256^{i rr}; the fold replaces it by w_N^{(256 i + j) rr}
            return wN((256 * i + jj) * rr) * np.exp(2j * np.pi * (i * rr) / 256)
        out[jj] = _stockham(Y[jj], [16, 16], tw_in)
    X = np.empty(N, complex)
    X[(j + S * np.arange(S)[None, :]).ravel()] = out.ravel()  # X[j + 256 k1] = Z[j][k1]
    ref = np.fft.fft(x)
    assert np.abs(X - ref).max() < 1e-8 * np.abs(ref).max()


@pytest.mark.parametrize("Q", [8, 16])
def test_c16_row_delivery_covers_every_element_once(Q):
    """Column phase thread (rl, ja) of CTA p holds Y[ja + 16 s][cols p + rl], s < 16; it sends it to
    CTA 16 s // cols, row 16 s % cols + ja: every (CTA, row, column) of the row phase exactly once,
    and the destination CTA owns row j = ja + 16 s."""
    cols = 256 // Q
    seen = np.zeros((Q, cols, 256), int)
    for p in range(Q):
        for rl in range(cols):
            for ja in range(16):
                for s in range(16):
                    dst, row = 16 * s // cols, 16 * s % cols + ja
                    j = ja + 16 * s
                    assert dst == j // cols and row == j % cols
                    seen[dst, row, p * cols + rl] += 1
    assert (seen == 1).all()
