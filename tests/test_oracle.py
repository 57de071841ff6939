"""Pins for the CPU oracle (T0).  No GPU needed.

Every check here ties oracle/ to something other than itself: the paper's printed
Eq. 1 factors and Listing 1 input (tests/golden/), closed forms of the DFT,
textbook invariants, brute force on tiny inputs, and numpy.fft (pocketfft, the
library family the paper compared against).
"""
import math
import os

import numpy as np
import pytest

import oracle
from oracle import dense
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_eq1():
    mats, name, rows = {}, None, []
    for line in open(os.path.join(GOLDEN, "eq1_dft4.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line.endswith(":"):
            if name:
                mats[name] = np.array(rows, dtype=np.complex128)
            name, rows = line[:-1], []
        else:
            rows.append([complex(t) for t in line.split()])
    mats[name] = np.array(rows, dtype=np.complex128)
    return mats


def _read_listing1():
    d = {}
    for line in open(os.path.join(GOLDEN, "listing1.txt")):
        if line.startswith("#") or ":" not in line:
            continue
        k, v = line.split(":", 1)
        d[k.strip()] = np.array([complex(t) for t in v.split()], dtype=np.complex128)
    return d


def c64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex64))


# ---------------------------------------------------------------- Eq. 1 / Eq. 2
def test_eq1_factors_match_paper():
    """each dense generator equals the printed factor, entry for entry."""
    g = _read_eq1()
    assert np.array_equal(dense.kron(dense.dft_matrix(2), dense.identity(2)).round(15), g["DFT2_kron_I2"])
    assert np.allclose(dense.twiddle(4, 2), g["D"], atol=1e-16)
    assert np.array_equal(dense.kron(dense.identity(2), dense.dft_matrix(2)).round(15), g["I2_kron_DFT2"])
    assert np.array_equal(dense.stride_perm(4, 2), g["Pi"])


def test_eq1_product_is_dft4():
    """the printed product equals DFT_4 -- and equals O1 applied column by column."""
    g = _read_eq1()
    prod = g["DFT2_kron_I2"] @ g["D"] @ g["I2_kron_DFT2"] @ g["Pi"]
    assert np.abs(prod - dense.dft_matrix(4)).max() < 1e-15
    cols = oracle.dft_naive(c64(np.eye(4)), -1)  # row t = DFT of e_t = column t of DFT_4
    assert np.abs(cols.T - prod).max() < 1e-15
    cols2 = oracle.fft_ct(c64(np.eye(4)), -1)
    assert np.abs(cols2.T - prod).max() < 1e-15


@pytest.mark.parametrize("N", [n for n in range(2, 65)])
def test_eq2_identity_all_splits(N):
    """P:73 Eq. 2 is an identity for every N = MK <= 64 (pins D and Pi conventions)."""
    for K in range(2, N):
        if N % K == 0:
            assert np.abs(dense.eq2_chain(N, K) - dense.dft_matrix(N)).max() < 1e-10


def test_eq2_transposed_readings_fail():
    """The other readings of D^N_M / Pi^N_K are not identities (so the pin discriminates)."""
    N, K = 8, 2
    M = N // K
    F = dense.dft_matrix(N)
    wrong_d = (dense.kron(dense.dft_matrix(K), dense.identity(M)) @ dense.twiddle(N, K)
               @ dense.kron(dense.identity(K), dense.dft_matrix(M)) @ dense.stride_perm(N, K))
    wrong_p = (dense.kron(dense.dft_matrix(K), dense.identity(M)) @ dense.twiddle(N, M)
               @ dense.kron(dense.identity(K), dense.dft_matrix(M)) @ dense.stride_perm(N, M))
    assert np.abs(wrong_d - F).max() > 0.5
    assert np.abs(wrong_p - F).max() > 0.5


@pytest.mark.parametrize("N", [4, 6, 8, 12, 30, 60])
def test_o2_equals_eq2_chain(N):
    """O2 (recursive Eq. 2) equals the dense Eq. 2 product applied to x."""
    x = synth.uniform_c64(N, 3, seed=5)
    p = min(q for q in range(2, N + 1) if N % q == 0)
    y_dense = (dense.eq2_chain(N, p) @ x.astype(np.complex128).T).T
    assert np.abs(oracle.fft_ct(x) - y_dense).max() < 1e-12


def test_listing1():
    """P:108-114 Listing 1 input; output derived by hand (golden)."""
    g = _read_listing1()
    x = c64(g["input"])[None]
    for y in (oracle.dft_naive(x), oracle.fft_ct(x)):
        assert np.abs(y[0] - g["output"]).max() < 1e-12
    y_dense = dense.eq2_chain(4, 2) @ g["input"]
    assert np.abs(y_dense - g["output"]).max() < 1e-12


# ---------------------------------------------------------------- closed forms
SIZES = [1, 2, 3, 4, 5, 7, 8, 60, 64, 105, 4096]


@pytest.mark.parametrize("N", SIZES)
@pytest.mark.parametrize("fn", ["naive", "ct"])
def test_closed_forms(N, fn):
    f = oracle.dft_naive if fn == "naive" else oracle.fft_ct
    # delta at n=0 -> all ones, exactly
    d = np.zeros((1, N), np.complex64); d[0, 0] = 1
    assert np.array_equal(f(d, -1)[0], np.ones(N, np.complex128))
    # zero -> exactly zero
    assert np.array_equal(f(np.zeros((1, N), np.complex64), -1)[0], np.zeros(N))
    # constant c -> N c at bin 0, ~0 elsewhere
    c = np.complex64(0.25 - 0.5j)
    y = f(np.full((1, N), c, np.complex64), -1)[0]
    assert abs(y[0] - N * complex(c)) <= 1e-12 * N
    if N > 1:
        assert np.abs(y[1:]).max() <= 1e-12 * N
    # tone x[n] = exp(+2 pi i k0 n / N) with sign -1 -> N delta_{k,k0}; sign +1 -> bin N-k0.
    # x is rounded to fp32 (|err| <= 2^-24 |x| per component), so ||Y - N delta||_2 <= N * 2^-23.
    if N > 1:
        k0 = (3 * N) // 7 % N or 1
        n = np.arange(N)
        tone = np.exp(2j * np.pi * ((k0 * n) % N) / N).astype(np.complex64)[None]
        ref = np.zeros(N); ref[k0] = N
        assert np.linalg.norm(f(tone, -1)[0] - ref) <= N * 2.0 ** -22
        ref2 = np.zeros(N); ref2[(N - k0) % N] = N
        assert np.linalg.norm(f(tone, +1)[0] - ref2) <= N * 2.0 ** -22


# ---------------------------------------------------------------- brute force / library
CROSS = [8, 16, 60, 64, 105, 210, 1000, 2187, 3125, 4096, 11, 13, 51, 4097, 2048, 512, 7, 49]


@pytest.mark.parametrize("N", CROSS)
@pytest.mark.parametrize("sign", [-1, 1])
def test_o2_vs_o1_vs_numpy(N, sign):
    x = synth.uniform_c64(N, 3, seed=N)
    y1 = oracle.dft_naive(x, sign)
    y2 = oracle.fft_ct(x, sign)
    xd = x.astype(np.complex128)
    yn = np.fft.fft(xd, axis=-1) if sign == -1 else np.fft.ifft(xd, axis=-1) * N
    assert oracle.rel_l2(y2, y1).max() <= 1e-13
    assert oracle.rel_l2(y1, yn).max() <= 1e-13
    assert oracle.rel_l2(y2, yn).max() <= 1e-13


def test_paper_protocol_p217():
    """random inputs, N = 32..1024, |result - numpy| / N < 1e-7 on every run."""
    for N in [32, 64, 128, 256, 512, 1024]:
        for trial in range(10):
            x = synth.uniform_c64(N, 1, seed=1000 * N + trial)
            y = oracle.fft_ct(x)
            yn = np.fft.fft(x.astype(np.complex128))
            assert np.abs(y - yn).max() / N < 1e-7


def test_spot_bin_matches_o1():
    N = 1000
    x = synth.uniform_c64(N, 1, seed=7)
    y = oracle.dft_naive(x)[0]
    for k in [0, 1, 17, 500, 999]:
        assert abs(oracle.spot_bin(x, k) - y[k]) <= 1e-12 * N


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("N", [8, 12, 60, 105, 128, 3125])
def test_invariants(N):
    x = synth.uniform_c64(N, 2, seed=N + 1)
    y = oracle.fft_ct(x)
    xd = x.astype(np.complex128)
    # Parseval: sum |Y|^2 = N sum |X|^2
    assert abs(np.sum(np.abs(y) ** 2) - N * np.sum(np.abs(xd) ** 2)) <= 1e-12 * N * np.sum(np.abs(xd) ** 2)
    # linearity (in double): F(a x0 + x1) = a F(x0) + F(x1)
    a = 0.3 - 1.7j
    z = a * xd[0] + xd[1]
    assert oracle.rel_l2(oracle.fft_ct_f64(z)[0], a * y[0] + y[1]).max() < 1e-13
    # Hermitian symmetry for real x: Y[N-k] = conj Y[k]
    xr = x.real.astype(np.float32).astype(np.complex64)
    yr = oracle.fft_ct(xr)
    k = np.arange(1, N)
    assert np.abs(yr[:, N - k] - np.conj(yr[:, k])).max() <= 1e-12 * N
    # shift theorem: x[(n - s) mod N] -> Y[k] w_N^{k s}
    s = 3
    ys = oracle.fft_ct(np.roll(x, s, axis=-1))
    kk = np.arange(N)
    assert np.abs(ys - y * np.exp(-2j * np.pi * kk * s / N)).max() <= 1e-12 * N
    # round trip: F^{-1}(F x) = N x
    back = oracle.fft_ct_f64(y, +1)
    assert np.abs(back - N * xd).max() <= 1e-12 * N


def test_scaled_unitarity_small():
    for N in [2, 3, 5, 6, 16, 30]:
        F = oracle.dft_naive(c64(np.eye(N)), -1).T
        assert np.abs(F @ F.conj().T - N * np.eye(N)).max() < 1e-10


def test_determinism():
    x = synth.uniform_c64(3125, 4, seed=3)
    a = oracle.fft_ct(x)
    b = oracle.fft_ct(x, nthreads=1)
    assert np.array_equal(a, b)


def test_tolerance_values():
    assert abs(oracle.tolerance(8) - 6e-6) < 1e-18
    assert abs(oracle.tolerance(4096) - 2.4e-5) < 1e-18
    assert abs(oracle.tolerance(3125) - 2.322e-5) < 1e-8
    assert oracle.tolerance(1) == 0.0


# ---------------------------------------------------------------- the gate metric itself
def test_rel_l2_hand_values():
    """oracle.rel_l2 against values computed by hand (BASELINE.json gate: per-transform
    ||y - y_ref||_2 / ||y_ref||_2).  Row 0: y = [3+4i, 0], ref = [0, 5]: the difference is
    [3+4i, -5], |.|^2 = 25 + 25 = 50, ||ref|| = 5 -> sqrt(50)/5 = sqrt(2) exactly."""
    e = oracle.rel_l2(np.array([[3 + 4j, 0]]), np.array([[0, 5]]))
    assert e.shape == (1,)
    assert abs(e[0] - math.sqrt(2.0)) < 1e-15
    # a pure phase error of pi/3 on every bin: |1 - e^{i pi/3}| = 2 sin(pi/6) = 1 -> exactly 1
    ref = np.array([[1 + 1j, -2 + 0.5j, 3j, 0.25]])
    e = oracle.rel_l2(ref * np.exp(1j * math.pi / 3), ref)
    assert abs(e[0] - 1.0) < 1e-15
    # sqrt, not the squared ratio: y = 2 ref -> 1 (squared would also be 1), y = 3 ref -> 2 (not 4)
    assert abs(oracle.rel_l2(3 * ref, ref)[0] - 2.0) < 1e-15
    # an error in the imaginary part only is counted: ref = [1, 1], y = [1, 1+i] -> 1/sqrt(2)
    e = oracle.rel_l2(np.array([[1, 1 + 1j]]), np.array([[1, 1]]))
    assert abs(e[0] - 1 / math.sqrt(2.0)) < 1e-15


def test_rel_l2_is_per_row():
    """One value per transform, not a whole-buffer norm: a wrong row next to exact rows
    keeps its own error (a global norm would dilute 1.0 to 1/sqrt(3) here)."""
    ref = np.array([[1, 0, 0], [0, 2, 0], [0, 0, 3]], dtype=np.complex128)
    y = ref.copy()
    y[1, 1] = 4  # row 1: |4 - 2| / 2 = 1
    e = oracle.rel_l2(y, ref)
    assert e.shape == (3,)
    assert e[0] == 0.0 and e[2] == 0.0
    assert abs(e[1] - 1.0) < 1e-15
    assert e.max() == e[1]


def test_rel_l2_zero_reference_and_dtypes():
    # zero reference row: the absolute L2 of y (nothing to divide by), exact zero for y = 0
    e = oracle.rel_l2(np.array([[0, 0], [3, 4j]]), np.zeros((2, 2)))
    assert e[0] == 0.0 and abs(e[1] - 5.0) < 1e-15
    # the GPU's complex64 output is upcast exactly before the difference: 1 + 2^-20 is exact in fp32
    y = np.array([[1 + 2.0 ** -20]], dtype=np.complex64)
    assert abs(oracle.rel_l2(y, np.array([[1.0]]))[0] - 2.0 ** -20) < 1e-22
    # a 1-D pair is one transform
    assert oracle.rel_l2(np.array([1, 1j]), np.array([1, 0])).shape == (1,)


def test_gate_negative_controls_cpu():
    """The gate accepts a correct fp32 FFT and rejects plausible wrong outputs.
    Correct: numpy's single-precision FFT (pocketfft, float32) of the same input.  Wrong: one bin
    perturbed by 10*tol*||y||, the conjugated spectrum, two bins swapped, the inverse's output."""
    for N in (64, 1000, 4096):
        x = synth.uniform_c64(N, 4, seed=7)
        ref = oracle.fft_ct(x, -1)
        tol = oracle.tolerance(N)
        good = np.fft.fft(x.astype(np.complex64), axis=1).astype(np.complex64)
        assert oracle.rel_l2(good, ref).max() <= tol
        bad = good.copy()
        bad[2, 5] += 10 * tol * np.linalg.norm(good[2])
        assert oracle.rel_l2(bad, ref).max() > tol
        assert oracle.rel_l2(np.conj(good), ref).max() > tol
        sw = good.copy()
        sw[:, [3, 7]] = sw[:, [7, 3]]
        assert oracle.rel_l2(sw, ref).max() > tol
        assert oracle.rel_l2(oracle.fft_ct(x, +1), ref).max() > tol
