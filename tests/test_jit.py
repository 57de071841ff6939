"""JIT mode: sizes with prime factors above 7.

CPU: the generated source compiles with NVRTC for sm_100a (no device needed), the
planner rejects what the JIT cannot do.  GPU: parity of the JIT kernels against the
oracle (whose recursive Cooley-Tukey falls back to the definition for prime lengths).
"""
import numpy as np
import pytest

import oracle
import synth

import paper_2207_06803_b200 as fftc

JIT_SIZES = [11, 13, 17, 19, 22, 23, 26, 29, 31, 33, 37, 41, 43, 47, 53, 59, 61, 121, 143, 169, 187, 253, 429,
             704, 1331, 2 * 61 * 29, 3328, 16 * 11 * 23, 11 * 13 * 17]


def _jit(N):
    return fftc.fftc_jit_source(N) is not None


@pytest.mark.parametrize("N", [11, 13, 61, 143, 3328, 2 * 61 * 29])
def test_jit_source_compiles_for_sm100a(N):
    r, log = fftc.fftc_jit_compile(N)
    assert r > 0, log


@pytest.mark.parametrize("L", [11, 61, 100, 125, 143, 243, 256, 2 * 61])
def test_jit_pass_source_compiles_for_sm100a(L):
    r, log = fftc.fftc_jit_pass_compile(L)
    assert r > 0, log


def test_jit_planner_domain():
    for N in JIT_SIZES:
        assert _jit(N), N
    assert not _jit(67)            # prime above 61
    assert not _jit(64 * 67)
    assert not _jit(1)
    assert fftc.fftc_jit_source(4096 * 11) is None  # above the single-pass limit (runtime passes)


def test_generated_codelet_source_shape():
    src = fftc.fftc_jit_source(13 * 16)
    assert "dft13" in src and "dft16" in src and "fftc_jit" in src
    assert "sm_" not in src  # architecture comes from the NVRTC options, not the source


@pytest.mark.gpu
@pytest.mark.parametrize("N", JIT_SIZES)
def test_gpu_jit_parity(N):
    torch = pytest.importorskip("torch")
    batch = 37
    x = synth.uniform_c64(N, batch, seed=N)
    for sign in (-1, 1):
        with fftc.Plan(N, batch, sign) as p:
            assert "kind=jit" in p.describe(), p.describe()
            y = p(torch.from_numpy(x).cuda())
            torch.cuda.synchronize()
            y = y.cpu().numpy()
        err = oracle.rel_l2(y, oracle.fft_ct(x, sign)).max()
        assert err <= min(oracle.tolerance(N), 2e-6), (N, sign, err)


@pytest.mark.gpu
def test_gpu_jit_unsupported():
    pytest.importorskip("torch")
    for N in (67, 64 * 67, 4096 * 67):
        with pytest.raises(fftc.FFTCError) as e:
            fftc.Plan(N, 2, -1)
        assert e.value.status == fftc.FFTC_ERROR_UNSUPPORTED_SIZE


LARGE_JIT = [(11 * 4096, 3), (13 * 13 * 256, 3), (61 * 1024, 2), (11 * 13 * 17 * 19, 2), (3 ** 5 * 59, 4),
             (11 * (1 << 16), 1)]


@pytest.mark.gpu
@pytest.mark.parametrize("N,batch", LARGE_JIT)
def test_gpu_jit_large_passes(N, batch):
    """N > 4096 with prime factors 11..61: runtime passes, each an NVRTC kernel specialised to
    its length (any radix from the emitter), both signs, against the oracle."""
    torch = pytest.importorskip("torch")
    x = synth.uniform_c64(N, batch, seed=N % 997)
    for sign in (-1, 1):
        with fftc.Plan(N, batch, sign) as p:
            assert "kind=gpass" in p.describe() and "jit" in p.describe(), p.describe()
            y = p(torch.from_numpy(x).cuda())
            torch.cuda.synchronize()
            y = y.cpu().numpy()
        err = oracle.rel_l2(y, oracle.fft_ct(x, sign)).max()
        assert err <= min(oracle.tolerance(N), 2e-6), (N, sign, err)


@pytest.mark.gpu
@pytest.mark.parametrize("N", [12288, 59049, 100000])
def test_gpu_gpass_compiled_kernel_without_jit(N, monkeypatch):
    """FFTC_GPASS_JIT=0: the compiled runtime-schedule pass kernel (k_gpass) stays correct."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("FFTC_GPASS_JIT", "0")
    x = synth.uniform_c64(N, 2, seed=N % 991)
    with fftc.Plan(N, 2, -1) as p:
        assert "kind=gpass" in p.describe() and "jit" not in p.describe(), p.describe()
        y = p(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        y = y.cpu().numpy()
    err = oracle.rel_l2(y, oracle.fft_ct(x, -1)).max()
    assert err <= min(oracle.tolerance(N), 2e-6), (N, err)



def _geo(src):
    import re
    m = re.search(r"constexpr int L = (\d+), LP = (\d+), COLS = (\d+), T = (\d+)", src)
    return tuple(int(v) for v in m.groups())


@pytest.mark.parametrize("L", [16, 27, 49, 81, 96, 100, 121, 125, 128, 176, 192, 243, 250, 256, 320, 343, 400, 512,
                               1024, 2048, 4096])
def test_jit_pass_geometry(L):
    """The generated pass kernel's tile geometry: an odd pitch >= L, <= 100 KB of shared memory,
    whole warps; the fused variant's T = COLS * L / R_0 (each thread one stage-0 butterfly)."""
    src = fftc.fftc_jit_pass_source(L)
    assert src, L
    L_, LP, COLS, T = _geo(src)
    assert L_ == L and LP % 2 == 1 and LP >= L
    assert COLS * LP * 8 <= 100 * 1024
    assert T % 32 == 0 and 32 <= T <= 512
    if "fused pass" in src:
        import re
        R0 = int(re.search(r"R0 = (\d+)", src).group(1))
        assert T == COLS * (L // R0)


@pytest.mark.gpu
@pytest.mark.parametrize("N,batch", [(6561, 3), (12288, 5), (11 * 4096, 2)])
def test_gpu_jit_pass_generic_variant(N, batch, monkeypatch):
    """FFTC_JIT_PASS_GENERIC=1: the non-fused generated pass kernel (staged load / store through
    shared memory) stays correct, both signs."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("FFTC_JIT_PASS_GENERIC", "1")
    x = synth.uniform_c64(N, batch, seed=N % 983)
    for sign in (-1, 1):
        with fftc.Plan(N, batch, sign) as p:
            y = p(torch.from_numpy(x).cuda())
            torch.cuda.synchronize()
            y = y.cpu().numpy()
        err = oracle.rel_l2(y, oracle.fft_ct(x, sign)).max()
        assert err <= min(oracle.tolerance(N), 2e-6), (N, sign, err)


@pytest.mark.gpu
@pytest.mark.parametrize("N,lens", [(1 << 21, "2048,1024"), (1 << 22, "4096,1024"), (3 * (1 << 20), "4096,768")])
def test_gpu_jit_long_passes(N, lens, monkeypatch):
    """Generated passes up to 4096 long (FFTC_LARGE=gpass FFTC_GPASS_LENGTHS: the fused kernel on
    2- and 4-column tiles), both signs, against the oracle."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("FFTC_LARGE", "gpass")
    monkeypatch.setenv("FFTC_GPASS_LENGTHS", lens)
    x = synth.uniform_c64(N, 2, seed=5)
    for sign in (-1, 1):
        with fftc.Plan(N, 2, sign) as p:
            assert "passes=" + lens.split(",")[0] in p.describe(), p.describe()
            y = p(torch.from_numpy(x).cuda())
            torch.cuda.synchronize()
            y = y.cpu().numpy()
        err = oracle.rel_l2(y, oracle.fft_ct(x, sign)).max()
        assert err <= min(oracle.tolerance(N), 2e-6), (N, sign, err)


@pytest.mark.gpu
@pytest.mark.parametrize("N,batch", [(143, 37), (1088, 5), (3328, 3)])
def test_gpu_jit_single_pass_generic_variant(N, batch, monkeypatch):
    """FFTC_JIT_GENERIC=1: the staged single-pass JIT kernel (the fused one is the default for
    N with two or more stages) stays correct, both signs, ragged last tile."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("FFTC_JIT_GENERIC", "1")
    x = synth.uniform_c64(N, batch, seed=N % 977)
    for sign in (-1, 1):
        with fftc.Plan(N, batch, sign) as p:
            assert "kind=jit" in p.describe(), p.describe()
            y = p(torch.from_numpy(x).cuda())
            torch.cuda.synchronize()
            y = y.cpu().numpy()
        err = oracle.rel_l2(y, oracle.dft_naive(x, sign)).max()
        assert err <= min(oracle.tolerance(N), 2e-6), (N, sign, err)
