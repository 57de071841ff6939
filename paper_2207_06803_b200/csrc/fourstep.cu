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
#include "fused.cuh"
#include "fourstep.h"

namespace fftc {

namespace {

// Pass 1: columns.  P: Sched<M, ..., TPF, C, F_FAST>; f = column within the tile.
template <class P, int MINB>
__global__ void __launch_bounds__(P::THREADS, MINB)
    k_cols(const float2* __restrict__ in, float2* __restrict__ work, const float2* __restrict__ tw,
           const float2* __restrict__ twA, const float2* __restrict__ twB, int K, long long N, float csign) {
  extern __shared__ float2 sm[];
  int f, lt;
  P::thread_coords(threadIdx.x, f, lt);
  const int tiles = K / P::FPB;
  const long long b = blockIdx.x / tiles;
  const int c = (blockIdx.x % tiles) * P::FPB + f;  // global column r
  const float2* gi = in + b * N + c;
  float2* go = work + b * N + c;
  run_stages<P, true, true>(
      sm, f, lt, true, tw,
      [&](int i) {
        float2 a = __ldcs(gi + (long long)i * K);
        return make_float2(a.x, csign * a.y);
      },
      [&](int j, float2 v) {
        const int e = c * j;  // < N <= 2^31
        const float2 w = cmul(__ldg(twA + (e & 4095)), __ldg(twB + (e >> 12)));
        go[(long long)j * K] = cmul(v, w);
      });
}

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
      sm, f, lt, true, tw, [&](int i) { return __ldcs(gi + i); }, [&](int, float2) {});
  __syncthreads();  // the transposed store reads rows written by other warps
  // X[j + M k1] for j in [j0, j0 + FPB): FPB contiguous outputs per k1.
  float2* go = out + b * N + j0;
  static_assert(FPB % 2 == 0, "row tile must hold an even number of rows");
  constexpr int HP = FPB / 2;
  constexpr int PAIRS = K * HP;
  for (int e = threadIdx.x; e < PAIRS; e += P::THREADS) {
    const int fp = 2 * (e % HP);
    const int k1 = e / HP;
    const float2 a = sm[P::sidx(fp, k1)];
    const float2 v = sm[P::sidx(fp + 1, k1)];
    __stcs(reinterpret_cast<float4*>(go + (long long)M * k1 + fp),
           make_float4(a.x, csign * a.y, v.x, csign * v.y));
  }
}

template <class P, int MINB>
cudaError_t launch_cols(const float2* in, float2* work, const float2* tw, const float2* twA,
                        const float2* twB, int K, long long N, long long batch, int conj, cudaStream_t st) {
  auto kern = k_cols<P, MINB>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long grid = batch * (K / P::FPB);
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)grid, P::THREADS, P::SMEM, st>>>(in, work, tw, twA, twB, K, N, conj ? -1.f : 1.f);
  return cudaGetLastError();
}

template <class P, int MINB>
cudaError_t launch_rows(const float2* work, float2* out, const float2* tw, int M, long long N, long long batch,
                        int conj, cudaStream_t st) {
  auto kern = k_rows<P, MINB>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long grid = batch * (M / P::FPB);
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)grid, P::THREADS, P::SMEM, st>>>(work, out, tw, M, N, conj ? -1.f : 1.f);
  return cudaGetLastError();
}

}  // namespace

#define FFTC_COL(M, RAD, TPF, C, MINB, ...) \
  {M, RAD::S, {__VA_ARGS__}, TPF, C, Sched<M, RAD, TPF, C, F_FAST>::SMEM, &launch_cols<Sched<M, RAD, TPF, C, F_FAST>, MINB>}
#define FFTC_ROW(K, RAD, TPF, FPB, PAD, MINB, ...)                                           \
  {K, RAD::S, {__VA_ARGS__}, TPF, FPB, Sched<K, RAD, TPF, FPB, LT_FAST, PAD>::SMEM,         \
   &launch_rows<Sched<K, RAD, TPF, FPB, LT_FAST, PAD>, MINB>}

using Rad_16x16 = Radices<16, 16>;
using Rad_16x16x16 = Radices<16, 16, 16>;
using Rad_32x32 = Radices<32, 32>;

static const ColEntry kCols[] = {
    FFTC_COL(256, Rad_16x16, 16, 16, 2, 16, 16),
    FFTC_COL(1024, Rad_32x32, 32, 8, 1, 32, 32),
    FFTC_COL(4096, Rad_16x16x16, 256, 4, 1, 16, 16, 16),
};
static const RowEntry kRows[] = {
    FFTC_ROW(256, Rad_16x16, 16, 32, 0, 1, 16, 16),
    FFTC_ROW(1024, Rad_32x32, 32, 8, 2, 1, 32, 32),
    FFTC_ROW(4096, Rad_16x16x16, 256, 4, 4, 1, 16, 16, 16),
};

const ColEntry* find_col(int M) {
  for (const auto& e : kCols)
    if (e.M == M) return &e;
  return nullptr;
}
const RowEntry* find_row(int K) {
  for (const auto& e : kRows)
    if (e.K == K) return &e;
  return nullptr;
}
int col_count() { return (int)(sizeof(kCols) / sizeof(kCols[0])); }
int row_count() { return (int)(sizeof(kRows) / sizeof(kRows[0])); }
const ColEntry* col_at(int i) { return (i >= 0 && i < col_count()) ? &kCols[i] : nullptr; }
const RowEntry* row_at(int i) { return (i >= 0 && i < row_count()) ? &kRows[i] : nullptr; }

}  // namespace fftc
