"""Host emulation of the six-step chunk algebra of csrc/dist.cu (test infrastructure).

Runs the exact index maps of the CUDA path -- pack, three all-to-alls, the two
strided column DFTs (numpy stands in for the kernels), the D^N_M twiddle and the
unpack -- on one rank's slab, with the all-to-all supplied by the caller
(torch.distributed over gloo in tests/test_dist_host.py, or an in-process list
exchange).  The geometry (M, K, K1, K2) comes from libfftc's planner
(fftc_dist_split), so the emulation follows the split the GPU would use.
"""
import numpy as np


def six_step_rank(x_p, N, P, p, split, a2a, sign=-1):
    """x_p: complex128 slab of rank p (N/P elements). a2a(send[P, chunk]) -> recv[P, chunk]."""
    M, K, K1, K2 = split
    Mp, Kp = M // P, K // P
    f = np.fft.fft if sign == -1 else (lambda a, axis=-1: np.fft.ifft(a, axis=axis) * a.shape[axis])
    # 1. pack: send[d][ql][rl] = x_p[ql K + d Kp + rl]
    send = x_p.reshape(Mp, P, Kp).transpose(1, 0, 2).copy()
    # 2. a2a #1 -> recv[s][ql][rl] = B[s Mp + ql][p Kp + rl] ; B = M x Kp
    B = a2a(send.reshape(P, -1)).reshape(M, Kp)
    # 3. DFT_M down columns, twiddle w_N^{(p Kp + rl) j}, transposed into send[d][rl][jl]
    Y = f(B, axis=0)  # Y[j][rl]
    j = np.arange(M)[:, None]
    r = p * Kp + np.arange(Kp)[None, :]
    Y = Y * np.exp(sign * 2j * np.pi * ((r * j) % N) / N)
    send = Y.reshape(P, Mp, Kp).transpose(0, 2, 1).copy()  # [d][rl][jl]
    # 4. a2a #2 -> V[r][jl] (K x Mp)
    V = a2a(send.reshape(P, -1)).reshape(K, Mp)
    # 5. DFT_K down columns jl (K2 > 1: Eq. 2 again, K = K1 K2)
    if K2 == 1:
        Z = f(V, axis=0)  # Z[k1][jl]
    else:
        W = V.reshape(K1, K2, Mp)                     # W[a][b][jl] = v[a K2 + b]
        W = f(W, axis=0)                              # DFT_K1 over a -> [ja][b][jl]
        ja = np.arange(K1)[:, None, None]
        b = np.arange(K2)[None, :, None]
        W = W * np.exp(sign * 2j * np.pi * ((b * ja) % K) / K)
        W = f(W, axis=1)                              # DFT_K2 over b -> [ja][kb][jl]
        Z = W.transpose(1, 0, 2).reshape(K, Mp)       # k = ja + K1 kb
    # 6. a2a #3 -> recv[s][k1l][jl]
    R = a2a(Z.reshape(P, -1)).reshape(P, Kp, Mp)
    # 7. unpack: X_p[k1l M + s Mp + jl] = recv[s][k1l][jl]
    return R.transpose(1, 0, 2).reshape(-1).copy()
