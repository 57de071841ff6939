// direct_tc.cu -- the paper's "direct DFT" as a batched dense product on tcgen05 tensor cores
// (product path, opt-in: fftc_plan_create_direct).
//
// Besides its recursive Cooley-Tukey factorizations, the paper evaluates the plain DFT as
// one dense matrix-vector product, y = DFT_N x (the "direct" curve of its
// evaluation).  For a batch of transforms that is a GEMM: with x interleaved
// (re, im) fp32, the rows of the [batch][2N] input times the real 2N x 2N matrix G,
//     G[2m][2k] = c, G[2m+1][2k] = -s, G[2m][2k+1] = s, G[2m+1][2k+1] = c,
//     c + i s = w^{mk}, w = exp(sign 2 pi i / N)      (exponent reduced mod N in integers)
// give the interleaved output rows: Y = X G, no de-interleaving.  On sm_100a it runs as
// tcgen05.mma kind::tf32 (M = 128 transforms per tile, N = K = 2N), accumulating in TMEM.
// TF32 keeps 10 mantissa bits, so the fp32 operands are split, x = x_hi + x_lo and
// G = G_hi + G_lo (hi = TF32-rounded), and the product is x_hi G_hi + x_hi G_lo + x_lo G_hi
// (3xTF32; the dropped x_lo G_lo is ~2^-22 relative) -- fp32-level accuracy from the
// tensor cores.  Per tile: one TMA tensor load of the [128][2N] fp32 rows (128-byte swizzle,
// the canonical K-major UMMA layout), an in-place hi/lo split into a second buffer, 3 x 2N/8
// MMAs issued by one thread, tcgen05.ld of the accumulator rows, a TMA tensor store.
// G_hi / G_lo are built on the host in double and stored in global memory already in the
// swizzled shared-memory image, so a CTA fetches them with one bulk copy.
#include <cuda.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "direct_tc.h"
#include "launch_util.h"
#include "tma.cuh"

namespace fftc {

namespace {

constexpr int kTileM = 128;

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// K-major, 128-byte-swizzle UMMA shared-memory descriptor (SBO = 8 rows x 128 B)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)1 << 16;                         // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;               // stride byte offset: 8-row core-matrix groups
  d |= (uint64_t)1 << 46;                         // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                         // layout: SWIZZLE_128B
  return d;
}

template <int N2>
__device__ __forceinline__ constexpr uint32_t instr_desc() {
  return (1u << 4)                     // D format: F32
         | (2u << 7) | (2u << 10)      // A, B format: TF32
         | ((uint32_t)(N2 >> 3) << 17)  // N
         | ((uint32_t)(kTileM >> 4) << 24);  // M = 128
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

// One CTA = 4 warps; tile = 128 transforms x 2N floats; persistent over tiles.
// Shared memory: X[kStages] (input tile -> TF32 hi in place -> output staging) | A_lo | G_hi | G_lo,
// each [2N/32 atoms][rows][128 B] with the 128-byte swizzle.  The TMA load of tile i + kStages-1
// is in flight while tile i is split, multiplied and stored.
template <int N, int kStages>
__global__ void __launch_bounds__(128, 1)
    k_direct_tc(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                const float* __restrict__ g_img, long long batch) {
  constexpr int N2 = 2 * N;                 // GEMM K and N
  constexpr int ATOMS = N2 / 32;            // 128-byte K atoms
  constexpr uint32_t A_BYTES = kTileM * N2 * 4;
  constexpr uint32_t G_BYTES = N2 * N2 * 4;
  constexpr uint32_t TMEM_COLS = N2 < 32 ? 32 : N2;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* base = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  float* Alo = reinterpret_cast<float*>(base + kStages * A_BYTES);
  unsigned char* G = base + (kStages + 1) * A_BYTES;  // G_hi then G_lo
  __shared__ __align__(8) uint64_t bar_g, bar_full[kStages], bar_mma;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long T = (batch + kTileM - 1) / kTileM;
  auto tile_of = [&](long long i) { return (long long)blockIdx.x + i * gridDim.x; };
  auto issue = [&](long long i) {  // TMA load of this CTA's i-th tile into stage i % kStages
    const long long t = tile_of(i);
    if (t >= T) return;
    unsigned char* X = base + (i % kStages) * A_BYTES;
    mbar_arrive_expect_tx(&bar_full[i % kStages], A_BYTES);
    for (int a = 0; a < ATOMS; ++a) tma_load_2d(X + a * (kTileM * 128), &tin, a * 32, (int)(t * kTileM), &bar_full[i % kStages]);
  };

  if (threadIdx.x == 0) {
    mbar_init(&bar_g, 1);
    for (int s = 0; s < kStages; ++s) mbar_init(&bar_full[s], 1);
    mbar_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive_expect_tx(&bar_g, 2 * G_BYTES);
    bulk_g2s(G, g_img, 2 * G_BYTES, &bar_g);
    for (int i = 0; i < kStages - 1; ++i) issue(i);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  constexpr uint32_t idesc = instr_desc<N2>();
  const uint32_t sAlo = smem_u32(Alo), sGhi = smem_u32(G), sGlo = smem_u32(G + G_BYTES);
  mbar_wait(&bar_g, 0);
  for (long long i = 0; tile_of(i) < T; ++i) {
    const long long t = tile_of(i);
    const int s = (int)(i % kStages);
    unsigned char* X = base + s * A_BYTES;
    const uint32_t sX = smem_u32(X);
    if (kStages == 1 && threadIdx.x == 0) {  // no prefetch: load this tile now
      bulk_wait_read0();
      issue(i);
    }
    mbar_wait(&bar_full[s], (uint32_t)((i / kStages) & 1));
    // hi / lo split (elementwise: the swizzled position is the same in both buffers)
    {
      float4* a4 = reinterpret_cast<float4*>(X);
      float4* l4 = reinterpret_cast<float4*>(Alo);
#pragma unroll 4
      for (int q = threadIdx.x; q < (int)(A_BYTES / 16); q += 128) {
        float4 v = a4[q];
        const float hx = __uint_as_float(to_tf32(v.x)), hy = __uint_as_float(to_tf32(v.y));
        const float hz = __uint_as_float(to_tf32(v.z)), hw = __uint_as_float(to_tf32(v.w));
        l4[q] = make_float4(v.x - hx, v.y - hy, v.z - hz, v.w - hw);
        a4[q] = make_float4(hx, hy, hz, hw);
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      // D = A_hi G_hi + A_hi G_lo + A_lo G_hi, K = 2N in steps of 8 (32 bytes within a 128-byte atom)
      for (int k = 0; k < N2 / 8; ++k) {
        const uint32_t off_a = (uint32_t)(k >> 2) * (kTileM * 128) + (uint32_t)(k & 3) * 32;
        const uint32_t off_g = (uint32_t)(k >> 2) * (N2 * 128) + (uint32_t)(k & 3) * 32;
        mma_tf32(tmem, umma_desc(sX + off_a), umma_desc(sGhi + off_g), idesc, k > 0);
        mma_tf32(tmem, umma_desc(sX + off_a), umma_desc(sGlo + off_g), idesc, 1);
        mma_tf32(tmem, umma_desc(sAlo + off_a), umma_desc(sGhi + off_g), idesc, 1);
      }
      mma_commit(&bar_mma);
      // refill the stage the previous tile used, once its store has finished reading it
      if (kStages > 1) {
        bulk_wait_read0();
        issue(i + kStages - 1);
      }
    }
    mbar_wait(&bar_mma, (uint32_t)(i & 1));
    tc_fence_after();
    // epilogue: warp w owns accumulator lanes (tile rows) 32w..32w+31; row r -> swizzled X
    {
      const int r = warp * 32 + lane;
      for (int c0 = 0; c0 < N2; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
        const int a = c0 / 32;
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // 16-byte chunks of the 128-byte row segment
          float4* dst = reinterpret_cast<float4*>(X + a * (kTileM * 128) + r * 128 + ((q ^ (r & 7)) << 4));
          *dst = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                             __uint_as_float(v[4 * q + 3]));
        }
      }
    }
    tc_fence_before();
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int a = 0; a < ATOMS; ++a) tma_store_2d(&tout, X + a * (kTileM * 128), a * 32, (int)(t * kTileM));
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait0();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
encode_fn get_encode() {
  static encode_fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (encode_fn)p;
  }
  return fn;
}
// [batch rows][2N floats] row-major, box [32 floats][128 rows], 128-byte swizzle
bool map_rows(CUtensorMap* m, const void* base, int N, long long batch) {
  encode_fn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)(2 * N), (cuuint64_t)batch};
  cuuint64_t strides[1] = {(cuuint64_t)(2 * N) * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)kTileM};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N, int S, int PER_SM>
cudaError_t launch_direct(const float2* in, float2* out, const float* g_img, long long batch, cudaStream_t st) {
  constexpr size_t smem = (size_t)(S + 1) * kTileM * 2 * N * 4 + (size_t)2 * (2 * N) * (2 * N) * 4 + 1024;
  static_assert(PER_SM * smem <= 227 * 1024, "CTAs per SM must fit in shared memory");
  auto kern = k_direct_tc<N, S>;
  // carveout 100: let PER_SM CTAs share an SM
  static PerDevice<KernelSetup> ks_pd;
  const KernelSetup& ks = ks_pd.get([&] { return kernel_setup(kern, 128, smem, 100, PER_SM); });
  if (ks.err != cudaSuccess) return ks.err;
  const int grid_max = ks.grid_max;
  CUtensorMap ti, to;
  if (!map_rows(&ti, in, N, batch) || !map_rows(&to, out, N, batch)) return cudaErrorInvalidValue;
  const long long T = (batch + kTileM - 1) / kTileM;
  if (T == 0) return cudaSuccess;
  long long gm = grid_max;
  if (const char* g = getenv("FFTC_DIRECT_GRID")) gm = atoll(g);  // tuning
  const unsigned grid = (unsigned)(T < gm ? T : gm);
  kern<<<grid, 128, smem, st>>>(ti, to, g_img, batch);
  return cudaGetLastError();
}

// host: round to TF32 (nearest, ties away from zero: cvt.rna)
float tf32_rna(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

}  // namespace

bool direct_supported(long long N) { return N == 16 || N == 32; }

// G_hi | G_lo in the swizzled K-major shared-memory image: element (j = output column,
// k = input column) of each at byte  (k/32) * (2N*128) + j*128 + (((k%32)/4 ^ (j%8)) * 16) + (k%4)*4
float* direct_tables(long long N, int sign, cudaError_t* err) {
  const int N2 = (int)(2 * N);
  std::vector<float> img((size_t)2 * N2 * N2, 0.f);
  for (int m = 0; m < (int)N; ++m)
    for (int kk = 0; kk < (int)N; ++kk) {
      const long long e = ((long long)m * kk) % N;
      const double a = 2.0 * M_PI * (double)e / (double)N;
      const double c = cos(a), s = sign * sin(a);
      // G[row k][col j]: rows = input (2m, 2m+1), cols = output (2kk, 2kk+1)
      const double g[2][2] = {{c, s}, {-s, c}};
      for (int u = 0; u < 2; ++u)
        for (int w = 0; w < 2; ++w) {
          const int k = 2 * m + u, j = 2 * kk + w;
          const float hi = tf32_rna((float)g[u][w]);
          const float lo = (float)(g[u][w] - (double)hi);
          const size_t off = (size_t)(k / 32) * (N2 * 128) + (size_t)j * 128 + (size_t)((((k % 32) / 4) ^ (j % 8)) * 16) +
                             (size_t)(k % 4) * 4;
          img[off / 4] = hi;
          img[(size_t)N2 * N2 + off / 4] = lo;
        }
    }
  float* d = nullptr;
  *err = cudaMalloc(&d, img.size() * sizeof(float));
  if (*err != cudaSuccess) return nullptr;
  *err = cudaMemcpy(d, img.data(), img.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (*err != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  return d;
}

cudaError_t direct_execute(long long N, const float2* in, float2* out, const float* g_img, long long batch,
                           cudaStream_t st) {
  if (batch == 0) return cudaSuccess;
  // measured on B200 (profiles/r01f): N = 16: 3-stage ring, 2 CTAs/SM (73 KB each) 5.6 TB/s;
  // N = 32: 3-stage ring, 1 CTA/SM (161 KB) 4.55 TB/s (1 stage x 2 CTAs/SM: 4.1 TB/s)
  if (N == 16) return launch_direct<16, 3, 2>(in, out, g_img, batch, st);
  if (N == 32) return launch_direct<32, 3, 1>(in, out, g_img, batch, st);
  return cudaErrorInvalidValue;
}

}  // namespace fftc
