// genstage.cuh -- one runtime-radix Stockham butterfly (product path).
//
// One butterfly j of a Stockham stage (radix R, Ns = product of the earlier radices) of a
// DFT_N held contiguously at a (read) / b (write): one level of the paper's Eq. 2 (PAPER.md
// P:73) with (N -> Ns R, K -> R, M -> Ns):
//   v[r] = a[j + r N/R];  v[r] *= w_{Ns R}^{(j mod Ns) r};  v = DFT_R v;
//   b[(j div Ns) Ns R + (j mod Ns) + r Ns] = v[r]
// Used by the runtime-schedule kernels (generic.cu, gpass.cu).
#pragma once
#include "fused.cuh"

namespace fftc {

template <int R>
__device__ __forceinline__ void gen_butterfly(const float2* __restrict__ a, float2* __restrict__ b, int N,
                                              int Ns, int j, const float2* __restrict__ tw) {
  const int NB = N / R;
  float2 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = a[j + r * NB];
  const int m = j % Ns;
  if (Ns > 1) {
    const float2* t = tw + (Ns - 1) + m;
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(t + (r - 1) * Ns));
  }
  Codelet<R>::run(v);
  const int o = (j / Ns) * Ns * R + m;
#pragma unroll
  for (int r = 0; r < R; ++r) b[o + r * Ns] = v[r];
}

// Dispatch one butterfly on a runtime radix from the generic codelet set.
__device__ __forceinline__ void gen_butterfly_rt(int R, const float2* __restrict__ a, float2* __restrict__ b, int N,
                                                 int Ns, int j, const float2* __restrict__ tw) {
  switch (R) {
    case 2: gen_butterfly<2>(a, b, N, Ns, j, tw); break;
    case 3: gen_butterfly<3>(a, b, N, Ns, j, tw); break;
    case 4: gen_butterfly<4>(a, b, N, Ns, j, tw); break;
    case 5: gen_butterfly<5>(a, b, N, Ns, j, tw); break;
    case 7: gen_butterfly<7>(a, b, N, Ns, j, tw); break;
    case 8: gen_butterfly<8>(a, b, N, Ns, j, tw); break;
    case 9: gen_butterfly<9>(a, b, N, Ns, j, tw); break;
    case 16: gen_butterfly<16>(a, b, N, Ns, j, tw); break;
    case 25: gen_butterfly<25>(a, b, N, Ns, j, tw); break;
    default: break;
  }
}

}  // namespace fftc
