"""The paper's direct DFT (the dense curve of P:231-235) as a batched GEMM on the
tcgen05 tensor cores (direct_tc.cu, 3xTF32), against the fp64 oracle."""
import numpy as np
import pytest

import oracle
import synth

import paper_2207_06803_b200 as fftc


@pytest.mark.gpu
@pytest.mark.parametrize("N", [16, 32])
@pytest.mark.parametrize("batch", [1, 127, 128, 129, 1000, 4096 + 37])
@pytest.mark.parametrize("sign", [-1, 1])
def test_direct_tc_parity(N, batch, sign):
    torch = pytest.importorskip("torch")
    x = synth.uniform_c64(N, batch, seed=N * 1000 + batch)
    with fftc.Plan.direct(N, batch, sign) as p:
        assert "kind=direct" in p.describe()
        y = p(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        y = y.cpu().numpy()
    err = oracle.rel_l2(y, oracle.dft_naive(x, sign)).max()
    # 3xTF32 keeps ~22 mantissa bits per product: fp32-level, within the BASELINE gate
    assert err <= min(oracle.tolerance(N), 2e-6), (N, batch, sign, err)


@pytest.mark.gpu
def test_direct_tc_special_inputs():
    torch = pytest.importorskip("torch")
    N, batch = 32, 256
    x = np.zeros((batch, N), np.complex64)
    x[:, 0] = 1.0                       # delta -> all ones
    x[1] = 0                            # zero row -> zeros
    x[2] = np.exp(-2j * np.pi * 5 * np.arange(N) / N * -1).astype(np.complex64)  # tone at k0 = 5
    with fftc.Plan.direct(N, batch, -1) as p:
        y = p(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.abs(y[0] - 1).max() < 1e-6
    assert np.abs(y[1]).max() == 0
    ref = np.zeros(N, np.complex128)
    ref[5] = N
    assert np.abs(y[2] - ref).max() < 1e-4


@pytest.mark.gpu
def test_direct_tc_rejects_other_sizes():
    pytest.importorskip("torch")
    for N in (8, 64, 60):
        with pytest.raises(fftc.FFTCError):
            fftc.Plan.direct(N, 4, -1)
