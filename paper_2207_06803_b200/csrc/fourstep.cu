// fourstep.cu -- two-pass large-N path (product path).
//
// Eq. 2 of PAPER.md applied once at the top with both factors large,
// N = M K, on the view A[q][r] = x[q K + r] (q < M rows, r < K columns):
//   pass 1 (k_cols): Pi^N_K + (I_K (x) DFT_M): a DFT_M down each column r
//                    (stride-K reads of C adjacent columns per CTA), then the
//                    D^N_M twiddle w_N^{r j}; writes W[j][r] (same strided layout).
//   pass 2 (k_rows): DFT_K (x) I_M: a DFT_K along each row j of W (contiguous),
//                    then the output index of Eq. 2, X[j + M k1], i.e. a
//                    transposed store staged through shared memory.
// Each inner DFT is itself a fused Stockham pass (fused.cuh).  Every element
// crosses HBM twice (read+write per pass): 32 B per complex element.
// The D^N_M twiddle w_N^e, e = r j < N, is read as A[e mod 4096] * B[e div 4096]
// (two fp32 tables built in double on the host, both L1/L2 resident).
#include <stdlib.h>
#include <string.h>

#include "colfft.cuh"
#include "fourstep.h"
#include "launch_util.h"

namespace fftc {

namespace {

// Pass 2: rows + transposed store.  P: Sched<K, ..., TPF, FPB, LT_FAST, PAD>.
template <class P, int MINB>
__global__ void __launch_bounds__(P::THREADS, MINB)
    k_rows(const float2* __restrict__ work, float2* __restrict__ out, const float2* __restrict__ tw, int M,
           long long N, float csign) {
  extern __shared__ float2 sm[];
  constexpr int K = P::N;
  constexpr int FPB = P::FPB;
  int f, lt;
  P::thread_coords(threadIdx.x, f, lt);
  const int tiles = M / FPB;
  const long long b = blockIdx.x / tiles;
  const int j0 = (blockIdx.x % tiles) * FPB;
  const float2* gi = work + b * N + (long long)(j0 + f) * K;
  run_stages<P, true, false>(
      sm, f, lt, true, tw, [&](int i, int) { return __ldcs(gi + i); }, [&](int, float2, int) {});
  __syncthreads();  // the transposed store reads rows written by other warps
  // X[j + M k1] for j in [j0, j0 + FPB): FPB contiguous outputs per k1; lanes walk j
  // (row stride SS chosen so a 16-lane phase hits 16 banks), 8-byte stores.
  float2* go = out + b * N + j0;
  constexpr int TOTAL = K * FPB;
  constexpr int PER = TOTAL / P::THREADS;
  static_assert(TOTAL % P::THREADS == 0, "tile must split evenly");
  sfor<PER>([&](auto n_) {
    constexpr int n = decltype(n_)::value;
    const int e = threadIdx.x + n * P::THREADS;
    const int fr = e % FPB, k1 = e / FPB;
    const float2 a = sm[P::sidx(fr, k1)];
    __stcs(go + (long long)M * k1 + fr, make_float2(a.x, csign * a.y));
  });
}

template <class P, int MINB>
cudaError_t launch_rows(const float2* work, float2* out, const float2* tw, int M, long long N, long long batch,
                        int conj, cudaStream_t st) {
  auto kern = k_rows<P, MINB>;
  static PerDevice<cudaError_t> attr_pd;
  const cudaError_t attr = attr_pd.get([&] {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
  });
  if (attr != cudaSuccess) return attr;
  const long long grid = batch * (M / P::FPB);
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)grid, P::THREADS, P::SMEM, st>>>(work, out, tw, M, N, conj ? -1.f : 1.f);
  return cudaGetLastError();
}

}  // namespace

#define FFTC_COL(NAME, M, RAD, TPF, C, LAY, MINB, ...)                                            \
  {M, RAD::S, {__VA_ARGS__}, TPF, C, Sched<M, RAD, TPF, C, F_FAST, 0, LAY>::SMEM,                 \
   Sched<M, RAD, TPF, C, F_FAST, 0, LAY_ODD>::SMEM, &launch_colx<Sched<M, RAD, TPF, C, F_FAST, 0, LAY>, false, MINB>, \
   &launch_colx<Sched<M, RAD, TPF, C, F_FAST, 0, LAY_ODD>, true, MINB>, NAME}
#define FFTC_ROW(NAME, K, RAD, TPF, FPB, PAD, MINB, ...)                                     \
  {K, RAD::S, {__VA_ARGS__}, TPF, FPB, Sched<K, RAD, TPF, FPB, LT_FAST, PAD>::SMEM,         \
   &launch_rows<Sched<K, RAD, TPF, FPB, LT_FAST, PAD>, MINB>, NAME}

using Rad_16x16 = Radices<16, 16>;
using Rad_16x32 = Radices<16, 32>;
using Rad_32x16 = Radices<32, 16>;
using Rad_8x16x16 = Radices<8, 16, 16>;
using Rad_16x16x8 = Radices<16, 16, 8>;
using Rad_16x16x4 = Radices<16, 16, 4>;
using Rad_16x16x16 = Radices<16, 16, 16>;
using Rad_32x32 = Radices<32, 32>;

// First entry per length = default; others are tuning candidates (FFTC_COL / FFTC_ROW = name).
static const ColEntry kCols[] = {
    FFTC_COL("c256_r16x16_t16x16", 256, Rad_16x16, 16, 16, LAY_FXOR, 2, 16, 16),
    FFTC_COL("c256_r16x16_t16x32", 256, Rad_16x16, 16, 32, LAY_FXOR, 1, 16, 16),
    FFTC_COL("c256_r16x16_t16x8", 256, Rad_16x16, 16, 8, LAY_INTER, 4, 16, 16),
    FFTC_COL("c512_r32x16_t16x8", 512, Rad_32x16, 16, 8, LAY_INTER, 2, 32, 16),
    FFTC_COL("c512_r16x32_t16x16", 512, Rad_16x32, 16, 16, LAY_FXOR, 1, 16, 32),
    FFTC_COL("c512_r32x16_t16x16", 512, Rad_32x16, 16, 16, LAY_FXOR, 1, 32, 16),
    FFTC_COL("c1024_r32x32_t32x8", 1024, Rad_32x32, 32, 8, LAY_INTER, 1, 32, 32),
    FFTC_COL("c1024_r32x32_t32x4", 1024, Rad_32x32, 32, 4, LAY_INTER, 2, 32, 32),
    FFTC_COL("c1024_r32x32_t32x16", 1024, Rad_32x32, 32, 16, LAY_FXOR, 1, 32, 32),
    FFTC_COL("c1024_r16x16x4_t64x8", 1024, Rad_16x16x4, 64, 8, LAY_INTER, 1, 16, 16, 4),
    FFTC_COL("c2048_r8x16x16_t128x4", 2048, Rad_8x16x16, 128, 4, LAY_INTER, 1, 8, 16, 16),
    FFTC_COL("c2048_r16x16x8_t128x4", 2048, Rad_16x16x8, 128, 4, LAY_INTER, 1, 16, 16, 8),
    FFTC_COL("c2048_r16x16x8_t128x2", 2048, Rad_16x16x8, 128, 2, LAY_INTER, 2, 16, 16, 8),
    FFTC_COL("c4096_r16x16x16_t256x4", 4096, Rad_16x16x16, 256, 4, LAY_INTER, 1, 16, 16, 16),
    FFTC_COL("c4096_r16x16x16_t256x2", 4096, Rad_16x16x16, 256, 2, LAY_INTER, 2, 16, 16, 16),
    FFTC_COL("c4096_r16x16x16_t128x4", 4096, Rad_16x16x16, 128, 4, LAY_INTER, 1, 16, 16, 16),
};
static const RowEntry kRows[] = {
    FFTC_ROW("r256_r16x16_t16x8", 256, Rad_16x16, 16, 8, 2, 4, 16, 16),
    FFTC_ROW("r256_r16x16_t16x32", 256, Rad_16x16, 16, 32, 1, 1, 16, 16),
    FFTC_ROW("r256_r16x16_t16x16", 256, Rad_16x16, 16, 16, 1, 2, 16, 16),
    FFTC_ROW("r512_r32x16_t16x16", 512, Rad_32x16, 16, 16, 1, 2, 32, 16),
    FFTC_ROW("r1024_r32x32_t32x8", 1024, Rad_32x32, 32, 8, 2, 1, 32, 32),
    FFTC_ROW("r1024_r32x32_t32x4", 1024, Rad_32x32, 32, 4, 4, 2, 32, 32),
    FFTC_ROW("r1024_r32x32_t32x16", 1024, Rad_32x32, 32, 16, 1, 1, 32, 32),
    FFTC_ROW("r2048_r16x16x8_t128x4", 2048, Rad_16x16x8, 128, 4, 4, 2, 16, 16, 8),
    FFTC_ROW("r4096_r16x16x16_t256x4", 4096, Rad_16x16x16, 256, 4, 4, 1, 16, 16, 16),
    FFTC_ROW("r4096_r16x16x16_t256x2", 4096, Rad_16x16x16, 256, 2, 8, 2, 16, 16, 16),
    FFTC_ROW("r4096_r16x16x16_t128x4", 4096, Rad_16x16x16, 128, 4, 4, 2, 16, 16, 16),
};

const ColEntry* find_col(int M) {
  if (const char* want = getenv("FFTC_COL"))
    for (const auto& e : kCols)
      if (e.M == M && strcmp(e.name, want) == 0) return &e;
  for (const auto& e : kCols)
    if (e.M == M) return &e;
  return nullptr;
}
const RowEntry* find_row(int K) {
  if (const char* want = getenv("FFTC_ROW"))
    for (const auto& e : kRows)
      if (e.K == K && strcmp(e.name, want) == 0) return &e;
  for (const auto& e : kRows)
    if (e.K == K) return &e;
  return nullptr;
}
int col_count() { return (int)(sizeof(kCols) / sizeof(kCols[0])); }
int row_count() { return (int)(sizeof(kRows) / sizeof(kRows[0])); }
const ColEntry* col_at(int i) { return (i >= 0 && i < col_count()) ? &kCols[i] : nullptr; }
const RowEntry* row_at(int i) { return (i >= 0 && i < row_count()) ? &kRows[i] : nullptr; }

ColGeom fourstep_cols_geom(const ColEntry* c, long long N, long long K) {
  ColGeom g{};
  g.tiles = (int)(K / c->cols);
  g.in_g = N;
  g.in_s = K;
  g.out_g = N;
  g.out_c = 1;
  g.out_s = K;
  g.out_cs = 0;
  g.ocl = 62;
  g.tw = 1;
  g.tw_shift = 0;
  g.tw_off = 0;
  return g;
}

}  // namespace fftc
