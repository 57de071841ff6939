// gpass.cu -- runtime-schedule multi-pass path for any 7-smooth N > 4096 (product path).
//
// The compiled large-N kernels (passes.cu) cover powers of two.  Every other 7-smooth N
// above the single-pass limit runs here: N = L_0 L_1 ... L_{p-1} (each L_s <= 256, a
// product of generic codelet radices), one HBM pass per factor, each pass one level of
// the paper's Eq. 2 in Stockham form (SURVEY App. A.2 with radix -> L_s):
//   column c < N/L, Ns = L_0 ... L_{s-1}:
//     v[r]  = a[c + r N/L] * w_{Ns L}^{(c mod Ns) r}           (Pi folded into the read; D)
//     v     = DFT_L v          (runtime Stockham sub-stages over the generic radices)
//     b[(c div Ns) Ns L + (c mod Ns) + r Ns] = v[r]
// A CTA owns clamp(4096 / L, 16, 256) adjacent columns (ragged at the right edge):
// coalesced loads with lanes walking columns, the DFT_L's in shared memory (one padded row per column, ping-pong
// buffers), and stores with lanes walking columns (Ns > 1: 16 columns are adjacent in the
// output) or walking r (Ns = 1: a column's outputs are contiguous).  Plain loads/stores,
// not TMA: for odd N the row pitch N/L * 8 bytes is not a multiple of 16.
#include <stdlib.h>

#include <vector>

#include "colfft.cuh"
#include "genstage.cuh"
#include "gpass.h"
#include "launch_util.h"

namespace fftc {

namespace {

constexpr int kGpThreads = 256;
constexpr int kGpTile = 4096;  // elements per CTA tile: cols = clamp(4096 / L, 16, 256) columns (power of two)

__host__ __device__ inline int gpass_cols(int L) {
  int c = 16;
  while (c < 256 && 2 * c * L <= kGpTile) c *= 2;
  return c;
}

__global__ void __launch_bounds__(kGpThreads, 4)
    k_gpass(const float2* __restrict__ in, float2* __restrict__ out, GPassStage g, long long N, int tiles,
            float csign_in, float csign_out) {
  extern __shared__ float2 sm[];
  __shared__ int s_cq[256], s_cm[256], s_R[kMaxStages];
  const int L = g.L, LP = L + 1;  // odd column pitch: lanes walking columns hit distinct banks
  const int cols = gpass_cols(L), lc = __ffs(cols) - 1;
  const long long NB = N / L;
  const long long b = blockIdx.x / tiles;
  const long long c0 = (long long)(blockIdx.x % tiles) * cols;
  const int nc = (int)(NB - c0 < cols ? NB - c0 : cols);
  float2* A = sm;
  float2* B = sm + cols * LP;
  // per-column index arithmetic once, in 32 bits (c < N / L < 2^31)
  if (threadIdx.x < kMaxStages) s_R[threadIdx.x] = threadIdx.x < g.S ? g.R[threadIdx.x] : 1;
  for (int f = threadIdx.x; f < cols; f += kGpThreads) {
    const int c = (int)c0 + f;
    s_cq[f] = c / g.Ns;
    s_cm[f] = c - (c / g.Ns) * g.Ns;
  }
  __syncthreads();
  // stage in: lanes walk columns; input twiddle w_T^{(c mod Ns) r}, T = Ns L.  Eight
  // elements per thread per round: all loads first (memory-level parallelism), then the
  // twiddles and the shared-memory stores.
  const float2* gi = in + b * N + c0;
  constexpr int U = 8;
  for (int e0 = threadIdx.x; e0 < (L << lc); e0 += U * kGpThreads) {
    float2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kGpThreads;
      const int f = e & (cols - 1), r = e >> lc;
      v[u] = (e < (L << lc) && f < nc) ? __ldcs(gi + f + (long long)r * NB) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kGpThreads;
      const int f = e & (cols - 1), r = e >> lc;
      if (e < (L << lc) && f < nc) {
        float2 x = v[u];
        x.y *= csign_in;
        if (g.Ns > 1) x = cmul(x, root_lookup_s(g.twA, g.twB, (long long)s_cm[f] * r, g.tws));
        A[f * LP + r] = x;
      }
    }
  }
  __syncthreads();
  // DFT_L of each column: runtime Stockham sub-stages, ping-pong between A and B
  int ns = 1;
  for (int s = 0; s < g.S; ++s) {
    const int R = s_R[s];
    const int NBs = L / R;
    for (int q = threadIdx.x; q < nc * NBs; q += kGpThreads) {
      const int f = q / NBs, j = q - (q / NBs) * NBs;
      gen_butterfly_rt(R, A + f * LP, B + f * LP, L, ns, j, g.tw);
    }
    __syncthreads();
    float2* t = A;
    A = B;
    B = t;
    ns *= R;
  }
  // stage out
  float2* go = out + b * N;
  if (g.Ns == 1) {
    // column c's outputs are contiguous at c L + r: lanes walk r
    for (int e = threadIdx.x; e < nc * L; e += kGpThreads) {
      const int f = e / L, r = e - (e / L) * L;
      const float2 v = A[f * LP + r];
      __stcs(go + (c0 + f) * L + r, make_float2(v.x, csign_out * v.y));
    }
  } else {
    // lanes walk columns: adjacent columns are adjacent in the output (within an Ns block)
    for (int e = threadIdx.x; e < (L << lc); e += kGpThreads) {
      const int f = e & (cols - 1), r = e >> lc;
      if (f < nc) {
        const float2 v = A[f * LP + r];
        __stcs(go + ((long long)s_cq[f] * L + r) * g.Ns + s_cm[f], make_float2(v.x, csign_out * v.y));
      }
    }
  }
}

}  // namespace

int gpass_split(long long N, int* Ls, int max, int max_prime, int max_len) {
  if (N <= 4096) return -1;
  if (const char* fl = getenv("FFTC_GPASS_LENGTHS")) {  // tuning: explicit pass lengths, e.g. "4096,4096"
    int q = 0;
    long long prod = 1;
    for (const char* c = fl; *c && q < max;) {
      const int e = atoi(c);
      if (e < 2 || e > 4096) return -1;
      Ls[q++] = e;
      prod *= e;
      while (*c && *c != ',') ++c;
      if (*c == ',') ++c;
    }
    if (prod == N) return q;
  }
  std::vector<int> f;
  long long n = N;
  for (int p = max_prime; p >= 2; --p) {
    bool prime = true;
    for (int d = 2; d * d <= p; ++d) prime = prime && p % d;
    if (!prime) continue;
    while (n % p == 0) {
      f.push_back(p);
      n /= p;
    }
  }
  if (n != 1) return -1;
  // fewest passes: largest-first assignment of the prime factors to the group with the
  // smallest product, every group <= kGpassMaxL
  for (int p = 2; p <= max; ++p) {
    std::vector<long long> g((size_t)p, 1);
    bool ok = true;
    for (int x : f) {
      size_t best = 0;
      for (size_t i = 1; i < g.size(); ++i)
        if (g[i] < g[best]) best = i;
      if (g[best] * x > max_len) {
        ok = false;
        break;
      }
      g[best] *= x;
    }
    if (!ok) continue;
    std::vector<long long> s = g;
    for (size_t i = 0; i < s.size(); ++i)  // descending
      for (size_t j = i + 1; j < s.size(); ++j)
        if (s[j] > s[i]) {
          long long t = s[i];
          s[i] = s[j];
          s[j] = t;
        }
    for (int i = 0; i < p; ++i) Ls[i] = (int)s[(size_t)i];
    return p;
  }
  return -1;
}

cudaError_t gpass_execute(const GPassPlanData& d, const float2* in, float2* out, float2* work, long long batch,
                          int conj, cudaStream_t st) {
  static PerDevice<cudaError_t> attr_pd;
  const cudaError_t attr = attr_pd.get([&] {
    return cudaFuncSetAttribute(k_gpass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * 256 * 17 * sizeof(float2)));
  });
  if (attr != cudaSuccess) return attr;
  const float2* src = in;
  for (int s = 0; s < d.p; ++s) {
    float2* dst = ((d.p - 1 - s) % 2 == 0) ? out : work;  // the last pass lands in out
    const GPassStage& g = d.st[s];
    const long long NB = d.N / g.L;
    const int cols = gpass_cols(g.L);
    const int tiles = (int)((NB + cols - 1) / cols);
    const long long grid = batch * tiles;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
    if (g.jk) {  // the pass specialised to (L, radices) by NVRTC
      cudaError_t e = jit_pass_launch(g.jk, src, dst, g.tw, g.twA, g.twB, d.N, g.Ns, g.tws, batch,
                                      conj && s == 0, conj && s == d.p - 1, st);
      if (e != cudaSuccess) return e;
    } else if (grid > 0) {
      const size_t smem = (size_t)2 * cols * (g.L + 1) * sizeof(float2);
      k_gpass<<<(unsigned)grid, kGpThreads, smem, st>>>(src, dst, g, d.N, tiles, (conj && s == 0) ? -1.f : 1.f,
                                                          (conj && s == d.p - 1) ? -1.f : 1.f);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    src = dst;
  }
  return cudaSuccess;
}

}  // namespace fftc
