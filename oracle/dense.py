"""Dense matrix semantics of the paper's factors -- TEST INFRASTRUCTURE ONLY.

Each generator is the plain dense matrix the paper names; nothing here is on
the product path.  Used by tests/test_oracle.py to pin the readings of Eq. 1
and Eq. 2 (§Background) against the paper's printed DFT_4
factorization, and to cross-check O1/O2 on tiny sizes.

Readings:
  * DFT_N[m, n] = w_N^{mn}, w_N = exp(sign 2 pi i / N), sign=-1 forward.
  * D^N_M (twiddle(N, M)): diagonal, position b*M + j holds w_N^{b*j}, b < K, j < M.
  * Pi^N_K (stride_perm(N, K)): (Pi x)[r*M + q] = x[q*K + r], q < M, r < K.
  * A (x) B: entry (i*rB + u, j*cB + v) = A[i, j] * B[u, v] (Table 1).
"""
from __future__ import annotations

import math

import numpy as np


def _w(N: int, e: int, sign: int = -1) -> complex:
    """w_N^e from the reduced exponent (e mod N), per-entry cos/sin."""
    e %= N
    a = 2.0 * math.pi * e / N
    return complex(math.cos(a), sign * math.sin(a))


def dft_matrix(N: int, sign: int = -1) -> np.ndarray:
    """DFT_N[m, n] = w_N^{m n}."""
    F = np.empty((N, N), dtype=np.complex128)
    for m in range(N):
        for n in range(N):
            F[m, n] = _w(N, m * n, sign)
    return F


def identity(n: int) -> np.ndarray:
    """I_n (P:62 'where the I is the identity matrix')."""
    return np.eye(n, dtype=np.complex128)


def twiddle(N: int, M: int, sign: int = -1) -> np.ndarray:
    """D^N_M: diag position b*M + j -> w_N^{b j}."""
    if N % M:
        raise ValueError("twiddle(N, M) requires M | N")
    K = N // M
    D = np.zeros((N, N), dtype=np.complex128)
    for b in range(K):
        for j in range(M):
            D[b * M + j, b * M + j] = _w(N, b * j, sign)
    return D


def stride_perm(N: int, K: int) -> np.ndarray:
    """Pi^N_K: (Pi x)[r*M + q] = x[q*K + r]."""
    if N % K:
        raise ValueError("stride_perm(N, K) requires K | N")
    M = N // K
    P = np.zeros((N, N), dtype=np.complex128)
    for r in range(K):
        for q in range(M):
            P[r * M + q, q * K + r] = 1.0
    return P


def kron(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Kronecker product written out: (A (x) B)[i*rB+u, j*cB+v] = A[i,j] B[u,v]."""
    ra, ca = A.shape
    rb, cb = B.shape
    out = np.zeros((ra * rb, ca * cb), dtype=np.complex128)
    for i in range(ra):
        for j in range(ca):
            out[i * rb:(i + 1) * rb, j * cb:(j + 1) * cb] = A[i, j] * B
    return out


def eq2_chain(N: int, K: int, sign: int = -1) -> np.ndarray:
    """(DFT_K (x) I_M) D^N_M (I_K (x) DFT_M) Pi^N_K with N = M K (Eq. 2)."""
    M = N // K
    return (kron(dft_matrix(K, sign), identity(M)) @ twiddle(N, M, sign)
            @ kron(identity(K), dft_matrix(M, sign)) @ stride_perm(N, K))
