"""FFTc factorization expressions (Listing 1, Table 1) -> radix schedule.

CPU tests of the product parser (`fftc_expr_radices`, host only).  The expressions the
tests feed it are first pinned, independently of the product, as identities: evaluated
densely with the oracle's factor generators (oracle/dense.py) they equal DFT_N.  GPU
parity of plans built from expressions is in `test_gpu_expr`.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from oracle import dense

import paper_2207_06803_b200 as fftc

LISTING1 = ("var result =  (DFT(2) ⊗ I(2)) · twiddle(4,2) ·\n"
            "              (I(2) ⊗ DFT(2)) · Permute(4,2) · InputComplex;")


def eq2_expr(radices, ascii_ops=False, with_matrix=True):
    """Recursive Eq. 2 expression for the Stockham radix list (innermost first) and its
    dense matrix (small N only): the outermost K = radices[-1], X_M = that of radices[:-1]."""
    kron, dot = ("&", "*") if ascii_ops else ("⊗", "·")
    if len(radices) == 1:
        n = radices[0]
        return "DFT(%d)" % n, (dense.dft_matrix(n) if with_matrix else None)
    K = radices[-1]
    M = math.prod(radices[:-1])
    N = K * M
    xs, xm = eq2_expr(radices[:-1], ascii_ops, with_matrix)
    s = "(DFT(%d) %s I(%d)) %s twiddle(%d,%d) %s (I(%d) %s (%s)) %s Permute(%d,%d)" % (
        K, kron, M, dot, N, M, dot, K, kron, xs, dot, N, K)
    if not with_matrix:
        return s, None
    mat = (dense.kron(dense.dft_matrix(K), dense.identity(M)) @ dense.twiddle(N, M)
           @ dense.kron(dense.identity(K), xm) @ dense.stride_perm(N, K))
    return s, mat


CASES = [[2, 2], [4, 4, 4], [8, 8], [4, 3, 5], [3, 5, 7], [2, 3, 5, 7], [5, 2], [7, 3, 2, 2]]


@pytest.mark.parametrize("radices", CASES)
def test_expression_is_an_identity_and_parses(radices):
    s, mat = eq2_expr(radices)
    N = math.prod(radices)
    # pin (independent of the product): the dense expression is DFT_N
    assert np.abs(mat - dense.dft_matrix(N)).max() < 1e-12
    assert fftc.fftc_expr_radices(s) == (N, radices)
    sa, _ = eq2_expr(radices, ascii_ops=True, with_matrix=False)
    assert fftc.fftc_expr_radices(sa) == (N, radices)


def test_listing1():
    """Listing 1 verbatim (var prefix, trailing input vector and ';'): N = 4, two radix-2
    stages; its dense value applied to the printed input gives the hand-derived output."""
    assert fftc.fftc_expr_radices(LISTING1) == (4, [2, 2])
    _, mat = eq2_expr([2, 2])
    x = np.array([1 + 1j, 2 + 2j, 3 + 3j, 4 + 4j])
    assert np.allclose(mat @ x, [10 + 10j, -4, -2 - 2j, -4j], atol=1e-12)


def test_bare_dft_leaves_the_planner_to_choose():
    assert fftc.fftc_expr_radices("DFT(4096)") == (4096, [])
    assert fftc.fftc_expr_radices("  DFT(60) ; ") == (60, [])


def test_factored_outer_dft_is_flattened():
    """(X_4 (x) I_2) with X_4 itself a factorization: stages = inner M then the K side."""
    x4, _ = eq2_expr([2, 2])
    s = "((%s) ⊗ I(2)) · twiddle(8,2) · (I(4) ⊗ DFT(2)) · Permute(8,4)" % x4
    assert fftc.fftc_expr_radices(s) == (8, [2, 2, 2])


def test_parenthesised_product_chain_is_flattened():
    s = "((DFT(2) ⊗ I(2)) · twiddle(4,2)) · ((I(2) ⊗ DFT(2)) · Permute(4,2))"
    assert fftc.fftc_expr_radices(s) == (4, [2, 2])


BAD = [
    # the transposed readings of D and Pi (the paper's N = 4 example cannot tell them apart;
    # at N = 8 they are not identities: SURVEY App. A.1) are rejected
    "(DFT(2) ⊗ I(4)) · twiddle(8,2) · (I(2) ⊗ DFT(4)) · Permute(8,2)",
    "(DFT(2) ⊗ I(4)) · twiddle(8,4) · (I(2) ⊗ DFT(4)) · Permute(8,4)",
    # factors out of order, wrong sizes, not a factorization
    "(I(2) ⊗ DFT(4)) · twiddle(8,4) · (DFT(2) ⊗ I(4)) · Permute(8,2)",
    "(DFT(2) ⊗ I(4)) · twiddle(8,4) · (I(2) ⊗ DFT(3)) · Permute(8,2)",
    "(DFT(2) ⊗ I(2)) · (I(2) ⊗ DFT(2)) · Permute(4,2)",
    "DFT(2) ⊗ I(2)",
    "I(4)",
    "DFT(4) ⊗",
    "foo(3)",
    "DFT(",
    "DFT(4) extra",
    "",
    "InputComplex",
    "(" * 100000 + "DFT(4)" + ")" * 100000,   # pathological nesting: rejected, no stack overflow
    "DFT(2)" + " ⊗ I(1)" * 100000,             # pathological Kronecker chain
    " · ".join(["I(2)"] * 100000),              # pathological product chain
]


@pytest.mark.parametrize("expr", BAD)
def test_rejects(expr):
    with pytest.raises(ValueError):
        fftc.fftc_expr_radices(expr)


def test_rejected_transposed_readings_are_not_identities():
    """Pin for the two rejections above: densely, those chains are not DFT_8."""
    K, M, N = 2, 4, 8
    a = (dense.kron(dense.dft_matrix(K), dense.identity(M)) @ dense.twiddle(N, K)
         @ dense.kron(dense.identity(K), dense.dft_matrix(M)) @ dense.stride_perm(N, K))
    b = (dense.kron(dense.dft_matrix(K), dense.identity(M)) @ dense.twiddle(N, M)
         @ dense.kron(dense.identity(K), dense.dft_matrix(M)) @ dense.stride_perm(N, M))
    F = dense.dft_matrix(N)
    assert np.abs(a - F).max() > 0.5 and np.abs(b - F).max() > 0.5


# ---------------------------------------------------------------- GPU parity
GPU_CASES = [[2, 2], [4, 4, 4], [8, 8], [4, 3, 5], [3, 5, 7], [2, 3, 5, 7], [8, 5, 5, 5], [16, 16, 16],
             [9, 9, 27], [2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2], [16, 16, 16, 4], [16, 16, 9, 9, 3],
             [7, 7, 7, 7, 7]]


@pytest.mark.gpu
@pytest.mark.parametrize("radices", GPU_CASES)
def test_gpu_expr(radices):
    """Plans built from FFTc expressions (fused if a compiled schedule has exactly these
    stages, else the runtime-schedule kernels) against the oracle, both signs."""
    torch = pytest.importorskip("torch")
    s, _ = eq2_expr(radices, with_matrix=False)
    N = math.prod(radices)
    batch = 5
    x = synth.uniform_c64(N, batch, seed=len(radices))
    for sign in (-1, 1):
        p = fftc.Plan.from_expr(s, batch, sign)
        try:
            d = p.describe()
            if N <= 4096 and ("kind=generic" in d or "kind=jit" in d):
                assert "radices=" + "x".join(map(str, radices)) in d, d
            y = p(torch.from_numpy(x).cuda())
            torch.cuda.synchronize()
            y = y.cpu().numpy()
        finally:
            p.close()
        err = oracle.rel_l2(y, oracle.fft_ct(x, sign)).max()
        assert err <= min(oracle.tolerance(N), 2e-6), (radices, sign, err, d)


# ---------------------------------------------------------------- property tests (hypothesis)
from hypothesis import given, settings, strategies as st  # noqa: E402


@settings(max_examples=200, deadline=None)
@given(st.lists(st.sampled_from([2, 3, 4, 5, 7, 8, 9, 16]), min_size=1, max_size=5), st.booleans())
def test_any_recursive_eq2_expression_round_trips(radices, ascii_ops):
    """Any right-recursive Eq. 2 expression parses back to its radix list (a lone DFT(n) is
    left to the planner)."""
    s, _ = eq2_expr(radices, ascii_ops=ascii_ops, with_matrix=False)
    want = radices if len(radices) > 1 else []
    assert fftc.fftc_expr_radices(s) == (math.prod(radices), want)


@settings(max_examples=300, deadline=None)
@given(st.lists(st.sampled_from([2, 3, 4, 5]), min_size=2, max_size=3), st.integers(0, 10 ** 6), st.integers(0, 4))
def test_mutated_expressions_fail_cleanly(radices, pos, kind):
    """Mutations of a valid expression (a dropped / swapped / altered character) either still
    parse to some valid schedule or raise ValueError -- never crash or hang the parser."""
    s, _ = eq2_expr(radices, with_matrix=False)
    i = pos % len(s)
    mut = [s[:i] + s[i + 1:], s[:i] + "(" + s[i:], s[:i] + ")" + s[i:], s[:i] + "9" + s[i + 1:],
           s.replace("I(", "DFT(", 1)][kind]
    try:
        N, R = fftc.fftc_expr_radices(mut)
        assert N >= 1 and (not R or math.prod(R) == N)
    except ValueError:
        pass
