"""CPU oracle for the batched 1D complex DFT -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product path
(``paper_2207_06803_b200`` / ``libfftc.so``) never imports it, and the two share
no code.

Functions (all fp64, see oracle/oracle.c for the paper citations):

* :func:`dft_naive`  -- O1, the definition Y[k] = sum_n X[n] w_N^{nk}
  (§Background).
* :func:`fft_ct`     -- O2, Eq. 2 applied recursively, smallest prime first
  (§Background Eq. 2).
* :func:`spot_bin`   -- one bin by O(N) direct summation (definition), for N=2^30.
* :func:`rel_l2`     -- the BASELINE.json gate metric (per-transform relative L2).

Inputs are numpy float32 arrays of shape (batch, N, 2) or complex64 (batch, N);
outputs are complex128 (batch, N).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (-O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, dp, fp, ip = ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int
        lib.oracle_dft_naive.argtypes = [fp, dp, i64, i64, ip, dp, i64]
        lib.oracle_dft_naive.restype = None
        lib.oracle_fft_ct.argtypes = [fp, dp, i64, i64, ip, ip]
        lib.oracle_fft_ct.restype = ctypes.c_int
        lib.oracle_fft_ct_f64.argtypes = [dp, dp, i64, i64, ip, ip]
        lib.oracle_fft_ct_f64.restype = ctypes.c_int
        lib.oracle_spot_bin.argtypes = [fp, i64, i64, ip, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double)]
        lib.oracle_spot_bin.restype = None
        lib.oracle_max_threads.argtypes = []
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _as_f32(x) -> np.ndarray:
    """(batch, N) complex64 or (batch, N, 2) float32 -> C-contiguous float32 (batch, N, 2)."""
    x = np.asarray(x)
    if np.iscomplexobj(x):
        if x.dtype != np.complex64:
            raise TypeError("oracle input must be the fp32 array the GPU receives (complex64)")
        x = x.view(np.float32).reshape(x.shape + (2,)) if x.ndim else x
    if x.dtype != np.float32 or x.shape[-1] != 2:
        raise TypeError("expected float32 (..., N, 2) or complex64 (..., N)")
    if x.ndim == 2:
        x = x[None]
    return np.ascontiguousarray(x)


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def dft_naive(x, sign: int = -1, idx=None) -> np.ndarray:
    """O1: naive O(N^2) DFT of transforms ``idx`` (default all). Returns complex128."""
    xf = _as_f32(x)
    batch, N = xf.shape[0], xf.shape[1]
    if idx is None:
        nt, ip = batch, None
    else:
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
        nt, ip = idx.size, idx.ctypes.data
    y = np.empty((nt, N), dtype=np.complex128)
    if nt and N:
        _load().oracle_dft_naive(xf.ctypes.data, y.ctypes.data, N, batch, int(sign), ip, nt)
    return y


def fft_ct(x, sign: int = -1, nthreads: int = 0) -> np.ndarray:
    """O2: recursive Cooley-Tukey per Eq. 2 (smallest prime first). Returns complex128."""
    xf = _as_f32(x)
    batch, N = xf.shape[0], xf.shape[1]
    y = np.empty((batch, N), dtype=np.complex128)
    if batch and N:
        rc = _load().oracle_fft_ct(xf.ctypes.data, y.ctypes.data, N, batch, int(sign), int(nthreads))
        if rc != 0:
            raise MemoryError("oracle_fft_ct: out of memory")
    return y


def fft_ct_f64(x, sign: int = -1, nthreads: int = 0) -> np.ndarray:
    """O2 on a complex128 input (batch, N)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    if x.ndim == 1:
        x = x[None]
    batch, N = x.shape
    y = np.empty_like(x)
    if batch and N:
        rc = _load().oracle_fft_ct_f64(x.ctypes.data, y.ctypes.data, N, batch, int(sign), int(nthreads))
        if rc != 0:
            raise MemoryError("oracle_fft_ct_f64: out of memory")
    return y


def spot_bin(x_row, k: int, sign: int = -1) -> complex:
    """Bin k of a single transform by direct O(N) summation (definition)."""
    xf = _as_f32(x_row)
    if xf.shape[0] != 1:
        raise ValueError("spot_bin takes one transform")
    N = xf.shape[1]
    re, im = ctypes.c_double(), ctypes.c_double()
    _load().oracle_spot_bin(xf.ctypes.data, N, int(k), int(sign), ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def rel_l2(y, y_ref) -> np.ndarray:
    """Per-transform ||y - y_ref||_2 / ||y_ref||_2, summed in double (BASELINE.json gate)."""
    y = np.asarray(y).astype(np.complex128, copy=False)
    y_ref = np.asarray(y_ref)
    if y.ndim == 1:
        y, y_ref = y[None], y_ref[None]
    num = np.sqrt(np.sum(np.abs(y - y_ref) ** 2, axis=-1))
    den = np.sqrt(np.sum(np.abs(y_ref) ** 2, axis=-1))
    out = np.where(den > 0, num / np.where(den > 0, den, 1.0), num)
    return out


def tolerance(N: int) -> float:
    """BASELINE.json gate: relative L2 <= 2e-6 * log2(N) (real log2; N=1 -> exact)."""
    import math
    return 2e-6 * math.log2(N) if N > 1 else 0.0
