// generic.cu -- runtime-schedule single-pass kernel (product path).
//
// Covers every N <= 4096 whose radix schedule uses the generic codelet set,
// for sizes without a compiled fast schedule (kernels_batch.cu).  Same Stockham
// stage as fused.cuh (one level of Eq. 2 per stage), but the
// stage list is a kernel argument, loops are runtime, and stages ping-pong
// between two shared-memory buffers.
#include "genstage.cuh"
#include "launch_util.h"
#include "registry.h"

namespace fftc {

namespace {

constexpr int kGenThreads = 256;

__global__ void __launch_bounds__(kGenThreads)
    k_generic(const float2* __restrict__ in, float2* __restrict__ out, const float2* __restrict__ tw,
              long long batch, float csign, GenericSched g, int fpb) {
  extern __shared__ float2 sm[];
  const int N = g.N;
  const long long f0 = (long long)blockIdx.x * fpb;
  const long long rem = batch - f0;
  const int nf = rem < fpb ? (int)rem : fpb;
  float2* A = sm;
  float2* B = sm + (size_t)fpb * N;
  const float2* gin = in + f0 * N;
  float2* gout = out + f0 * N;
  const int total = nf * N;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    float2 x = gin[e];
    A[e] = make_float2(x.x, csign * x.y);
  }
  __syncthreads();
  int Ns = 1;
  for (int s = 0; s < g.S; ++s) {
    const int R = g.R[s];
    const int NB = N / R;
    for (int q = threadIdx.x; q < nf * NB; q += blockDim.x) {
      const int f = q / NB, j = q % NB;
      const float2* a = A + (size_t)f * N;
      float2* b = B + (size_t)f * N;
      gen_butterfly_rt(R, a, b, N, Ns, j, tw);
    }
    __syncthreads();
    float2* t = A;
    A = B;
    B = t;
    Ns *= R;
  }
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    float2 x = A[e];
    gout[e] = make_float2(x.x, csign * x.y);
  }
}

}  // namespace

bool generic_supports_radix(int R) {
  switch (R) {
    case 2: case 3: case 4: case 5: case 7: case 8: case 9: case 16: case 25: return true;
    default: return false;
  }
}

cudaError_t launch_generic(const GenericSched& g, const float2* in, float2* out, const float2* tw,
                           long long batch, int conj, cudaStream_t st) {
  // transforms per CTA: fill ~32 KB of ping-pong buffers
  int fpb = (int)(2048 / g.N);
  if (fpb < 1) fpb = 1;
  const size_t smem = (size_t)2 * fpb * g.N * sizeof(float2);
  static PerDevice<cudaError_t> attr_pd;
  const cudaError_t attr = attr_pd.get([&] {
    return cudaFuncSetAttribute(k_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * kGenericMaxN * sizeof(float2)));
  });
  if (attr != cudaSuccess) return attr;
  const long long grid = (batch + fpb - 1) / fpb;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  k_generic<<<(unsigned)grid, kGenThreads, smem, st>>>(in, out, tw, batch, conj ? -1.0f : 1.0f, g, fpb);
  return cudaGetLastError();
}

}  // namespace fftc
