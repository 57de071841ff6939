// colfft.cuh -- strided "column" DFT_L kernel (product path).
//
// The large-N paths apply Eq. 2 at the top level with both factors
// large; each factor is a batch of DFT_L's along a strided axis of a 2D view
// ("columns").  k_colx computes DFT_L down C adjacent columns per CTA (columns are
// unit-stride apart, so a warp reads C*8-byte contiguous segments), with the inner
// DFT_L a fused Stockham pass (fused.cuh, F_FAST mapping: lanes walk columns).
//
// Geometry (runtime, ColGeom): column c = grp * G + ci (ci < G = tiles * C);
//   input  element i : in  + grp*in_g  + ci + i*in_s
//   output element k : out + grp*out_g + ci*out_c + (k >> ocl)*out_cs + (k & omask)*out_s
//   (or, with npeer > 0, peer[k >> ocl] + grp*out_g + ci*out_c + (k & omask)*out_s: the
//    chunk goes straight into another rank's receive buffer over NVLink)
//   optional twiddle : y_k *= w_T^{((ci >> tw_shift) + tw_off) * k}   (T-point root,
//                      read as A[e mod 4096] * B[e div 4096] from two fp32 tables)
// OUT_T = false: the last stage stores HBM directly (lanes walk columns; needs out_c = 1).
// OUT_T = true : the last stage stores shared memory, then a cooperative store walks k
//                (lanes walk the transform), for outputs whose columns are far apart
//                (the six-step's chunked layouts).
#pragma once
#include "colgeom.h"
#include "fused.cuh"

namespace fftc {


// w_T^e for 0 <= e < T from the two-level tables A[e mod 4096] * B[e div 4096]
__device__ __forceinline__ float2 root_lookup(const float2* __restrict__ A, const float2* __restrict__ B,
                                              long long e) {
  return cmul(__ldg(A + (e & 4095)), __ldg(B + (e >> 12)));
}
// the same with a balanced split (A: 2^sh entries w_T^t, B: w_T^{2^sh h}): both tables stay
// small enough to live in L1 next to the pass kernels' shared-memory tiles
__device__ __forceinline__ float2 root_lookup_s(const float2* __restrict__ A, const float2* __restrict__ B,
                                                long long e, int sh) {
  return cmul(__ldg(A + (e & ((1LL << sh) - 1))), __ldg(B + (e >> sh)));
}

template <class P, bool OUT_T, int MINB>
__global__ void __launch_bounds__(P::THREADS, MINB)
    k_colx(const float2* __restrict__ in, float2* __restrict__ out, const float2* __restrict__ tw,
           const float2* __restrict__ twA, const float2* __restrict__ twB, ColGeom g, float csign_in,
           float csign_out) {
  extern __shared__ float2 sm[];
  static_assert(P::MAP == F_FAST, "column kernel walks columns");
  constexpr int L = P::N;
  constexpr int C = P::FPB;
  constexpr int RL = P::R(P::S - 1);   // last-stage radix
  constexpr int NSL = P::ns(P::S - 1); // last-stage Ns: outputs k = j + r NSL
  constexpr int NB2 = ilog2(highbit(RL - 1)) + 1;  // powers w^(2^b) needed for r < RL
  int f, lt;
  P::thread_coords(threadIdx.x, f, lt);
  const long long grp = blockIdx.x / g.tiles;
  const int ci0 = (blockIdx.x % g.tiles) * C;
  const int ci = ci0 + f;
  const float2* gi = in + grp * g.in_g + ci;
  const long long omask = (1LL << g.ocl) - 1;
  // Output twiddle w_T^{c k}, c = (ci >> tw_shift) + tw_off.  In the last stage a thread's
  // outputs are k = j + r NSL: w^{c k} = w^{c j} (w^{c NSL})^r -- one table lookup per
  // butterfly for the base, the step powers w^{c NSL 2^b} once per thread, and at most
  // popcount(r) complex products per element (all from tables built in double).
  const long long ctw = g.tw ? (long long)(ci >> g.tw_shift) + g.tw_off : 0;
  float2 sp[NB2];
  if (g.tw) {
    sp[0] = root_lookup(twA, twB, ctw * NSL);
    sfor<NB2 - 1>([&](auto b_) {
      constexpr int b = decltype(b_)::value + 1;
      sp[b] = cmul(sp[b - 1], sp[b - 1]);
    });
  }
  float2 base = make_float2(1.f, 0.f);
  auto twiddle = [&](int k, float2 v, int r) {
    if (g.tw) {
      if (r == 0) base = root_lookup(twA, twB, ctw * k);
      float2 w = base;
      sfor<NB2>([&](auto b_) {
        constexpr int b = decltype(b_)::value;
        if (r & (1 << b)) w = cmul(w, sp[b]);
      });
      v = cmul(v, w);
    }
    return v;
  };
  auto load = [&](int i, int) {
    float2 a = __ldcs(gi + (long long)i * g.in_s);
    return make_float2(a.x, csign_in * a.y);
  };
  if constexpr (!OUT_T) {
    float2* go = out + grp * g.out_g + ci * g.out_c;
    run_stages<P, true, true>(sm, f, lt, true, tw, load, [&](int k, float2 v, int r) {
      v = twiddle(k, v, r);
      float2* dst = g.npeer ? reinterpret_cast<float2*>(g.peer[k >> g.ocl]) + grp * g.out_g + ci * g.out_c
                            : go + ((long long)k >> g.ocl) * g.out_cs;
      __stcs(dst + ((long long)k & omask) * g.out_s, make_float2(v.x, csign_out * v.y));
    });
  } else {
    // last stage: twiddled values back into the exchange buffer, then a store walking k
    run_stages<P, true, true, true>(sm, f, lt, true, tw, load,
                                    [&](int k, float2 v, int r) { sm[P::sidx(f, k)] = twiddle(k, v, r); });
    __syncthreads();
    float2* go = out + grp * g.out_g;
    constexpr int TOTAL = L * C;
    static_assert(TOTAL % P::THREADS == 0, "tile must split evenly");
    constexpr int PER = TOTAL / P::THREADS;
    sfor<PER>([&](auto n_) {
      constexpr int n = decltype(n_)::value;
      const int e = threadIdx.x + n * P::THREADS;
      const int k = e % L, cc = e / L;
      const float2 v = sm[P::sidx(cc, k)];
      float2* dst = g.npeer ? reinterpret_cast<float2*>(g.peer[k >> g.ocl]) + grp * g.out_g
                            : go + ((long long)k >> g.ocl) * g.out_cs;
      __stcs(dst + (long long)(ci0 + cc) * g.out_c + ((long long)k & omask) * g.out_s,
             make_float2(v.x, csign_out * v.y));
    });
  }
}

template <class P, bool OUT_T, int MINB>
static cudaError_t launch_colx(const float2* in, float2* out, const float2* tw, const float2* twA,
                               const float2* twB, const ColGeom& g, long long groups, int conj_in,
                               int conj_out, cudaStream_t st) {
  auto kern = k_colx<P, OUT_T, MINB>;
  static PerDevice<cudaError_t> attr_pd;
  const cudaError_t attr = attr_pd.get([&] {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
  });
  if (attr != cudaSuccess) return attr;
  const long long grid = groups * g.tiles;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)grid, P::THREADS, P::SMEM, st>>>(in, out, tw, twA, twB, g, conj_in ? -1.f : 1.f,
                                                    conj_out ? -1.f : 1.f);
  return cudaGetLastError();
}

}  // namespace fftc
