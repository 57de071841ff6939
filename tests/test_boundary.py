"""C-ABI boundary and host logic (CPU; no GPU needed).

* libfftc.so loads and exports every function declared in include/fftc.h.
* The planner (fftc_factorize / fftc_plan_split) obeys SURVEY §8(a) a1: product of
  radices = N, radices from the codelet set, deterministic, -1 for prime factors > 7.
* Without a device, plan creation fails loudly (NULL + FFTC_ERROR_NO_DEVICE) -- there
  is no CPU fallback.
"""
import math
import os
import re
import subprocess

import pytest

import paper_2207_06803_b200 as fftc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "fftc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fftc_[a-z_]+)\s*\(", txt)))


def test_library_exports_header_symbols():
    lib_path = fftc.LIB_PATH
    assert os.path.exists(lib_path), "libfftc.so must be built (build())"
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    declared = _header_functions()
    assert len(declared) >= 12
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    fftc.load()  # dlopen works without a GPU


def test_status_strings():
    for s in range(8):
        assert fftc.fftc_status_string(s).startswith("FFTC_")


def smooth7(n):
    for p in (2, 3, 5, 7):
        while n % p == 0:
            n //= p
    return n == 1


ALLOWED = {2, 3, 4, 5, 7, 8, 9, 10, 14, 15, 16, 25, 27, 30, 32}


@pytest.mark.parametrize("N", [n for n in range(1, 4097) if smooth7(n)])
def test_planner_single_pass(N):
    R = fftc.fftc_factorize(N)
    assert R is not None
    assert math.prod(R) == N
    assert all(r in ALLOWED for r in R)
    assert fftc.fftc_factorize(N) == R  # deterministic
    kind, M, K = fftc.fftc_plan_split(N)
    assert (kind, M, K) == (1, N, 1)


@pytest.mark.parametrize("N", [11, 13, 22, 4097, 17 * 64, 0, -5])
def test_planner_rejects(N):
    assert fftc.fftc_factorize(N) is None
    assert fftc.fftc_plan_split(N)[0] == -1


def test_planner_bench_sizes():
    # SURVEY §8(a) a1 examples (compiled schedules)
    assert fftc.fftc_factorize(4096) == [16, 16, 16]
    assert fftc.fftc_factorize(64) == [8, 8]
    assert fftc.fftc_factorize(60) == [4, 15]
    assert fftc.fftc_factorize(105) == [7, 15]
    for N in (8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 60, 105, 210, 1000, 2187, 3125):
        assert fftc.fftc_candidates(N), N  # a compiled fast schedule exists for every BASELINE size
    assert math.prod(fftc.fftc_factorize(2187)) == 2187
    assert math.prod(fftc.fftc_factorize(3125)) == 3125


@pytest.mark.parametrize("N,M,K", [(1 << 16, 256, 256), (1 << 20, 512, 2048), (1 << 24, 4096, 4096)])
def test_planner_fourstep_split(N, M, K):
    assert fftc.fftc_plan_split(N) == (2, M, K)
    assert math.prod(fftc.fftc_factorize(N)) == N


def test_planner_passes():
    for n in range(9, 41):
        Ls = fftc.fftc_plan_passes(1 << n)
        assert Ls is not None and math.prod(Ls) == 1 << n
        # 2^17..2^20: two passes of <= 1024, 2^21..2^23: two passes with 2048/4096-long ones,
        # 2^25..2^28: three (last 256); else ceil(n/8) of <= 256
        if n in (21, 22, 23):
            assert Ls == {21: [2048, 1024], 22: [4096, 1024], 23: [4096, 2048]}[n], (n, Ls)
            continue
        big = 17 <= n <= 20 or 25 <= n <= 28
        want = 2 if 17 <= n <= 20 else 3 if 25 <= n <= 28 else (n + 7) // 8
        if 25 <= n <= 28:
            assert Ls[-1] == 256
        assert len(Ls) == want, (n, Ls)
        assert all(16 <= L <= (1024 if big else 256) for L in Ls)
        assert Ls == sorted(Ls, reverse=True)
        if not 25 <= n <= 28:
            assert max(Ls) <= 2 * min(Ls)  # balanced
    assert fftc.fftc_plan_passes(3 * 4096) is None
    assert fftc.fftc_plan_passes(256) is None


def _smooth(n):
    for p in (2, 3, 5, 7):
        while n % p == 0:
            n //= p
    return n == 1


def test_planner_gpasses():
    """Runtime-schedule multi-pass split: product N, lengths <= 512 and 7-smooth, fewest
    passes (a lower bound is ceil(log_256 N)), longest first, deterministic."""
    sizes = [4097 - 1 + 3 * 2, 12288, 13122, 15625, 16807, 19683, 40960, 46656, 59049, 78125, 100000,
             248832, 10 ** 6, 3 ** 13, 3 ** 15, 5 ** 10, 7 ** 8, 6 ** 10]
    for N in sizes:
        if not _smooth(N):
            continue
        Ls = fftc.fftc_plan_gpasses(N)
        assert Ls is not None, N
        assert math.prod(Ls) == N and all(2 <= L <= 1024 and _smooth(L) for L in Ls), (N, Ls)
        assert len(Ls) >= math.ceil(math.log(N, 512) - 1e-12) and 2 <= len(Ls) <= 4
        assert Ls == sorted(Ls, reverse=True)
        assert Ls == fftc.fftc_plan_gpasses(N)
    assert fftc.fftc_plan_gpasses(3 ** 10) == [243, 243]
    assert fftc.fftc_plan_gpasses(4096) is None        # single pass
    assert fftc.fftc_plan_gpasses(11 * 4096) is None   # prime factor > 7
    assert fftc.fftc_plan_gpasses(257 * 257) is None   # prime 257
    assert fftc.fftc_plan_gpasses(10 ** 5) == [400, 250]  # JIT passes: up to 512 long


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = fftc.fftc_plan_create(64, 16, -1)
    assert h == 0
    assert fftc.fftc_last_error() == fftc.FFTC_ERROR_NO_DEVICE
    with pytest.raises(fftc.FFTCError):
        fftc.Plan(64, 16, -1)


def test_invalid_args_before_device():
    # argument validation precedes the device check
    assert fftc.fftc_plan_create(0, 1, -1) == 0
    assert fftc.fftc_last_error() == fftc.FFTC_ERROR_INVALID_VALUE
    assert fftc.fftc_plan_create(8, 1, 0) == 0
    assert fftc.fftc_last_error() == fftc.FFTC_ERROR_INVALID_VALUE
    assert fftc.fftc_plan_create(8, -1, -1) == 0
    assert fftc.fftc_last_error() == fftc.FFTC_ERROR_INVALID_VALUE
    assert fftc.fftc_plan_create(67, 1, -1) == 0  # prime > 61: neither compiled nor JIT codelets
    assert fftc.fftc_last_error() == fftc.FFTC_ERROR_UNSUPPORTED_SIZE
    assert fftc.fftc_plan_create(67 * 4096, 1, -1) == 0  # prime > 61 above the single-pass limit
    assert fftc.fftc_last_error() == fftc.FFTC_ERROR_UNSUPPORTED_SIZE
    assert fftc.fftc_execute(0, 0, 0, 0) == fftc.FFTC_ERROR_INVALID_VALUE


def test_default_schedules_follow_the_measured_policy():
    """The first candidate per N is the planner's default: paired-FP32 codelets exactly where
    they measured faster on B200, the scalar schedules elsewhere; the warp-shuffle
    exchange for N = 64 and L1::no_allocate stage-0 loads for 2048 / 4096 (DESIGN §6 K1)."""
    packed = {128, 105, 210, 1000, 3125, 2048}
    special = {64: "n64_r8x8_t8x8_shfl", 2048: "n2048_r16x16x8_t128x1_pk_na", 4096: "n4096_r16x16x16_t256x1_na",
               60: "n60_r4x15_t4x16"}
    for N in (8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 60, 105, 210, 1000, 2187, 3125):
        names = fftc.fftc_candidates(N)
        assert names, N
        assert ("_pk" in names[0]) == (N in packed), (N, names[0])
        if N in special:
            assert names[0] == special[N], (N, names[0])
        assert len(set(names)) == len(names), N
