// passes.cu -- multi-pass large-N path with TMA tensor tiles (product path).
//
// For N above the single-pass limit, N = L_0 L_1 ... L_{p-1} (each L_s <= 256) and the
// transform is p HBM passes, each one level of the paper's Eq. 2 applied
// at the pass level in Stockham autosort form (SURVEY App. A.2 with radix -> L_s):
//   pass s, Ns = L_0...L_{s-1}, NB = N / L_s columns c:
//     v[r]  = a[c + r NB]                                   (Pi folded into the column read)
//     v[r] *= w_{Ns L}^{(c mod Ns) r}          (s > 0)       (D^{Ns L}_{Ns})
//     v     = DFT_{L_s} v                                   (a fused Stockham pass, fused.cuh)
//     b[(c div Ns) Ns L + (c mod Ns) + r Ns] = v[r]         (natural order after the last pass)
// A CTA owns C = 16 adjacent columns (one 128-byte segment per row; C = 8, 64-byte rows,
// for L = 512 / 1024).  The [L rows][C cols] tile is fetched by ONE 3-D TMA tensor load
// (cp.async.bulk.tensor, 128B/64B-swizzled shared layout, completion on an mbarrier),
// transformed in place, and -- for s > 0 -- written back by ONE 4-D TMA tensor store
// (the autosort write is a [L][C] box of a
// (Ns, L, NB/Ns, batch) view).  Pass 0 (Ns = 1) writes each column's L outputs
// contiguously, via coalesced 8-byte stores.  CTAs are persistent with NBUF tile buffers:
// NBUF <= 2 refills a buffer right after its store has read it (the tile after next streams
// in while the current one is computed); NBUF >= 3 keeps NBUF - 1 loads ahead and refills the
// buffer of the PREVIOUS tile at the end of each iteration, so the issuing thread never
// waits on the store it has just committed.
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include "launch_util.h"
#include "passes.h"
#include "passtile.cuh"
#include "tma.cuh"

namespace fftc {

namespace {

template <class P, bool FIRST, int MINB, int NBUF>
__global__ void __launch_bounds__(P::THREADS, MINB)
    k_pass(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
           float2* __restrict__ out_first, const float2* __restrict__ tw, const float2* __restrict__ twA,
           const float2* __restrict__ twB, PassGeom g, float csign_in, float csign_out) {
  static_assert(NBUF >= 1 && NBUF <= 4, "one to four tile buffers");
  constexpr bool RING = NBUF >= 3;            // deferred refill (see the file header)
  constexpr int AHEAD = RING ? NBUF - 1 : NBUF;  // tiles issued before the first compute
  constexpr int L = P::N, C = P::FPB;
  constexpr uint32_t TILE_BYTES = (uint32_t)L * C * 8u;
  extern __shared__ __align__(1024) unsigned char smraw[];
  float2* buf0 = reinterpret_cast<float2*>(smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));
  __shared__ __align__(8) uint64_t full[NBUF];
  int f, lt;
  P::thread_coords(threadIdx.x, f, lt);
  const long long T = g.tiles_total;
  const int tpb = g.tiles_per_batch;
  constexpr int BOX = L < 256 ? L : 256;  // TMA boxes are at most 256 rows
  auto issue = [&](long long t, int k) {
    const int b = (int)(t / tpb), c0 = (int)(t % tpb) * C;
    mbar_arrive_expect_tx(&full[k], TILE_BYTES);
    sfor<L / BOX>([&](auto h_) {
      constexpr int h = decltype(h_)::value;
      tma_load_3d(buf0 + k * L * C + h * BOX * C, &tin, c0, h * BOX, b, &full[k]);
    });
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < NBUF; ++k) mbar_init(&full[k], 1);
  __syncthreads();
  // the CTA's it-th tile: groups of g.group adjacent tiles (their TMA rows share pages and DRAM
  // rows), groups dealt round-robin over the grid; group = 1 is the plain grid stride
  const int grp = g.group;
  auto tile_of = [&](int i) -> long long {
    return ((long long)(i / grp) * gridDim.x + blockIdx.x) * grp + (i % grp);
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < AHEAD; ++k)
      if (tile_of(k) < T) issue(tile_of(k), k);
  int it = 0;
  for (long long t = tile_of(0); t < T; t = tile_of(++it)) {
    const int k = it % NBUF;
    float2* sm = buf0 + k * L * C;
    const int b = (int)(t / tpb), c0 = (int)(t % tpb) * C;
    const int c = c0 + f;
    // one sub-stage-0 butterfly per thread: its input twiddles are formed under the TMA wait
    constexpr bool PRE = !FIRST && (L / P::R(0) <= P::TPF);
    PassTwPre pre{};
    if constexpr (PRE) pre = pass_tw_pre<P>(c, lt, g.Ns, twA, twB, g.tws);
    mbar_wait(&full[k], (it / NBUF) & 1);
    // first pass, 8-column tiles: one TMA store of the tile in the pass-0 output layout
    // (measured faster for L = 512/1024); 16-column tiles: coalesced 8-byte stores, lanes
    // walking each column's contiguous outputs (measured faster for L <= 256)
    constexpr bool TMA0 = FIRST && C == 8;
    pass_tile<P, !FIRST, TMA0>(sm, f, lt, c, g.Ns, tw, twA, twB, g.tws, csign_in, csign_out,
                               PRE ? &pre : nullptr);
    if constexpr (FIRST && !TMA0) {
      __syncthreads();
      pass0_store<P>(sm, out_first + (long long)b * g.N + (long long)c0 * L,
                     [](float2* q, float2 v) { __stcs(q, v); });
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0 && (!FIRST || TMA0)) {
      if constexpr (!FIRST) {
        sfor<L / BOX>([&](auto h_) {
          constexpr int h = decltype(h_)::value;
          tma_store_4d(&tout, sm + h * BOX * C, c0 % g.Ns, h * BOX, c0 / g.Ns, b);
        });
      } else {
        // pass 0: column c's outputs are contiguous at c L + k -- one box [16][C][L/16] of the
        // (k % 16, c, k / 16, batch) view
        tma_store_4d(&tout, sm, 0, c0, 0, b);
      }
      bulk_commit();
    }
    if constexpr (RING) {
      // refill the previous tile's buffer: its store (committed one iteration ago) has had a
      // whole tile of compute to read it; the store just committed may stay in flight
      if (threadIdx.x == 0 && tile_of(it + AHEAD) < T) {
        bulk_wait_read1();
        issue(tile_of(it + AHEAD), (it + AHEAD) % NBUF);
      }
    } else if (threadIdx.x == 0 && tile_of(it + NBUF) < T) {
      bulk_wait_read0();  // the store has finished reading this buffer
      issue(tile_of(it + NBUF), k);
    }
  }
  if (threadIdx.x == 0) bulk_wait0();
}

template <class P, int MINB, int NBUF>
cudaError_t launch_pass(bool first, const CUtensorMap& tin, const CUtensorMap& tout, float2* out_first,
                        const float2* tw, const float2* twA, const float2* twB, const PassGeom& g, int conj_in,
                        int conj_out, cudaStream_t st) {
  constexpr size_t smem = (size_t)NBUF * P::N * P::FPB * sizeof(float2) + 1024;
  auto kern = first ? k_pass<P, true, MINB, NBUF> : k_pass<P, false, MINB, NBUF>;
  static PerDevice<KernelSetup> ks_first_pd;
  const KernelSetup& ks_first = ks_first_pd.get([&] { return kernel_setup(k_pass<P, true, MINB, NBUF>, P::THREADS, smem); });
  static PerDevice<KernelSetup> ks_later_pd;
  const KernelSetup& ks_later = ks_later_pd.get([&] { return kernel_setup(k_pass<P, false, MINB, NBUF>, P::THREADS, smem); });
  const KernelSetup& ks = first ? ks_first : ks_later;
  if (ks.err != cudaSuccess) return ks.err;
  const int gm = ks.grid_max;
  if (g.tiles_total == 0) return cudaSuccess;
  const long long groups = (g.tiles_total + g.group - 1) / g.group;
  const unsigned grid = (unsigned)(groups < gm ? groups : gm);
  kern<<<grid, P::THREADS, smem, st>>>(tin, tout, out_first, tw, twA, twB, g, conj_in ? -1.f : 1.f,
                                      conj_out ? -1.f : 1.f);
  return cudaGetLastError();
}

}  // namespace

// C = 16 columns (128-byte rows, TMA 128B swizzle) for L <= 256; C = 8 (64-byte rows, 64B
// swizzle) for L = 512 / 1024 so a tile stays <= 64 KB.
#define FFTC_PASS(NAME, L, RAD, TPF, MINB, NBUF, ...)                                                    \
  {L, RAD::S, {__VA_ARGS__}, TPF, 16, &launch_pass<Sched<L, RAD, TPF, 16, F_FAST, 0, LAY_TMA128>, MINB, NBUF>, \
   NAME}
#define FFTC_PASS2(NAME, L, RAD, TPF, MINB, NBUF, ...)                                                  \
  {L, RAD::S, {__VA_ARGS__}, TPF, 2, &launch_pass<Sched<L, RAD, TPF, 2, F_FAST, 0, LAY_TMA16>, MINB, NBUF>, \
   NAME}
#define FFTC_PASS4(NAME, L, RAD, TPF, MINB, NBUF, ...)                                                  \
  {L, RAD::S, {__VA_ARGS__}, TPF, 4, &launch_pass<Sched<L, RAD, TPF, 4, F_FAST, 0, LAY_TMA16>, MINB, NBUF>, \
   NAME}
#define FFTC_PASS8(NAME, L, RAD, TPF, MINB, NBUF, ...)                                                  \
  {L, RAD::S, {__VA_ARGS__}, TPF, 8, &launch_pass<Sched<L, RAD, TPF, 8, F_FAST, 0, LAY_TMA64>, MINB, NBUF>, \
   NAME}

using PRad_4x4 = Radices<4, 4>;
using PRad_8x4 = Radices<8, 4>;
using PRad_8x8 = Radices<8, 8>;
using PRad_16x8 = Radices<16, 8>;
using PRad_16x16 = Radices<16, 16>;
using PRad_32x16 = Radices<32, 16>;
using PRad_16x32 = Radices<16, 32>;
using PRad_32x32 = Radices<32, 32>;
using PRad_16x16x8 = Radices<16, 16, 8>;
using PRad_16x16x16 = Radices<16, 16, 16>;

// First entry per length = default; FFTC_PASS=<name> pins a candidate (tuning).
static const PassEntry kPasses[] = {
    FFTC_PASS("p16_r4x4", 16, PRad_4x4, 4, 8, 2, 4, 4),
    FFTC_PASS("p32_r8x4", 32, PRad_8x4, 4, 8, 2, 8, 4),
    FFTC_PASS("p64_r8x8", 64, PRad_8x8, 8, 6, 2, 8, 8),
    FFTC_PASS("p64_r8x8_m4", 64, PRad_8x8, 8, 4, 2, 8, 8),
    FFTC_PASS("p128_r16x8", 128, PRad_16x8, 16, 3, 2, 16, 8),
    FFTC_PASS("p128_r16x8_b2m2", 128, PRad_16x8, 16, 2, 2, 16, 8),
    FFTC_PASS("p128_r16x8_b2m4", 128, PRad_16x8, 16, 4, 2, 16, 8),
    FFTC_PASS("p256_r16x16_b2m2", 256, PRad_16x16, 16, 2, 2, 16, 16),
    FFTC_PASS("p256_r16x16", 256, PRad_16x16, 16, 3, 2, 16, 16),
    FFTC_PASS("p256_r16x16_b2m1", 256, PRad_16x16, 16, 1, 2, 16, 16),
    FFTC_PASS("p256_r16x16_b1m4", 256, PRad_16x16, 16, 4, 1, 16, 16),
    FFTC_PASS("p256_r16x16_b3m2", 256, PRad_16x16, 16, 2, 3, 16, 16),
    FFTC_PASS("p128_r16x8_b3m4", 128, PRad_16x8, 16, 4, 3, 16, 8),
    FFTC_PASS("p128_r16x8_b4m3", 128, PRad_16x8, 16, 3, 4, 16, 8),
    FFTC_PASS8("p512_r16x32_c8t32", 512, PRad_16x32, 32, 2, 2, 16, 32),
    FFTC_PASS8("p512_r32x16_c8", 512, PRad_32x16, 16, 3, 2, 32, 16),
    FFTC_PASS8("p512_r32x16_c8m2", 512, PRad_32x16, 16, 2, 2, 32, 16),
    FFTC_PASS8("p512_r16x32_c8t32m1", 512, PRad_16x32, 32, 1, 2, 16, 32),
    FFTC_PASS8("p512_r16x32_c8t32b3", 512, PRad_16x32, 32, 2, 3, 16, 32),
    FFTC_PASS8("p1024_r32x32_c8b2", 1024, PRad_32x32, 32, 1, 2, 32, 32),
    FFTC_PASS8("p1024_r32x32_c8b1", 1024, PRad_32x32, 32, 3, 1, 32, 32),
    FFTC_PASS8("p1024_r32x32_c8b1m2", 1024, PRad_32x32, 32, 2, 1, 32, 32),
    FFTC_PASS8("p1024_r32x32_c8b3", 1024, PRad_32x32, 32, 1, 3, 32, 32),
    FFTC_PASS2("p2048_r16x16x8_c2b3", 2048, PRad_16x16x8, 128, 2, 3, 16, 16, 8),
    FFTC_PASS2("p4096_r16x16x16_c2b3", 4096, PRad_16x16x16, 256, 1, 3, 16, 16, 16),
    FFTC_PASS2("p4096_r16x16x16_c2b2", 4096, PRad_16x16x16, 256, 1, 2, 16, 16, 16),
    FFTC_PASS4("p2048_r16x16x8_c4b3", 2048, PRad_16x16x8, 128, 1, 3, 16, 16, 8),
    FFTC_PASS4("p4096_r16x16x16_c4b1", 4096, PRad_16x16x16, 128, 1, 1, 16, 16, 16),
    // a cluster of 4 CTAs per 8-column tile, each the 1024-point sub-DFT of one row residue class
    {4096, 2, {32, 32}, 32, 8, &launch_cpass4096, "cp4096_q4_r32x32_c8b2", 4},
    // the tile being computed in registers, 4 columns, next tile's TMA load in shared memory
    {4096, 3, {16, 16, 16}, 128, 4, &launch_rpass4096, "rp4096_r16x16x16_c4"},
};

// the entry of length L among a comma-separated list of candidate names
static const PassEntry* pass_named(int L, const char* names) {
  for (const auto& e : kPasses) {
    if (e.L != L) continue;
    const size_t n = strlen(e.name);
    for (const char* q = names; q && *q;) {
      const char* end = strchr(q, ',');
      const size_t len = end ? (size_t)(end - q) : strlen(q);
      if (len == n && strncmp(q, e.name, n) == 0) return &e;
      q = end ? end + 1 : nullptr;
    }
  }
  return nullptr;
}

const PassEntry* find_pass(int L, long long N, bool first) {
  if (first)
    if (const char* want = getenv("FFTC_PASS_FIRST"))
      if (const PassEntry* e = pass_named(L, want)) return e;
  if (const char* want = getenv("FFTC_PASS"))
    if (const PassEntry* e = pass_named(L, want)) return e;
  // measured on B200 (profiles/r01j, tools/pass_matrix.sh): the 3-buffer ring wins for every
  // 1024-long pass (2^20 1.58 -> 1.44 ms, 2^28 2.67 -> 2.62 ms), for the later 512-long passes
  // (2^18 1.49 -> 1.43 ms) and for the later 256-long passes of three-pass plans (N > 2^20:
  // 2^24 2.40 -> 2.35 ms) but not of two-pass ones (2^16 1.49 -> 1.53 ms, 2^17 1.52 ->
  // 1.58 ms); first passes of length <= 512 keep two buffers (no TMA store to wait for)
  const char* pick = nullptr;
  if (L == 1024) pick = "p1024_r32x32_c8b3";
  else if (L == 4096) pick = "rp4096_r16x16x16_c4";  // profiles/r02g: 2^22 1.90 -> 1.78, 2^23 2.11 -> 1.93 ms
  else if (L == 2048) pick = first ? "p2048_r16x16x8_c2b3" : "p2048_r16x16x8_c4b3";
  else if (L == 512 && !first) pick = "p512_r16x32_c8t32b3";
  else if (L == 256 && !first && N > (1LL << 20)) pick = "p256_r16x16_b3m2";
  if (pick)
    if (const PassEntry* e = pass_named(L, pick)) return e;
  for (const auto& e : kPasses)
    if (e.L == L) return &e;
  return nullptr;
}

// ---------------------------------------------------------------- host: tensor maps
typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static encode_fn get_encode() {
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

// shared layout of a tile row of C complex64 columns: 128 B (C = 16) and 64 B (C = 8) rows are
// TMA-swizzled, 16-byte rows (C = 2, the 2048/4096-long passes) are linear
static CUtensorMapSwizzle tile_swizzle(int C) {
  return C == 16 ? CU_TENSOR_MAP_SWIZZLE_128B : C == 8 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE;  // C = 2, 4
}

// in: a [batch][L rows][NB cols] view, box [C cols][min(L, 256) rows] (the TMA box limit)
static bool map_in(CUtensorMap* m, const void* base, long long N, int L, int C, long long batch) {
  encode_fn enc = get_encode();
  if (!enc) return false;
  const long long NB = N / L;
  cuuint64_t dims[3] = {(cuuint64_t)NB, (cuuint64_t)L, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)NB * 8, (cuuint64_t)N * 8};
  cuuint32_t box[3] = {(cuuint32_t)C, (cuuint32_t)(L < 256 ? L : 256), 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, tile_swizzle(C), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// cluster pass input: rows r = Q i + q of the [batch][L rows][NB cols] view as a (c, q, i, batch)
// view, box [C cols][1][256 rows][1] -- CTA q of a cluster loads only its residue class
static bool map_in_cluster(CUtensorMap* m, const void* base, long long N, int L, int C, int Q, long long batch) {
  encode_fn enc = get_encode();
  if (!enc) return false;
  const long long NB = N / L;
  cuuint64_t dims[4] = {(cuuint64_t)NB, (cuuint64_t)Q, (cuuint64_t)(L / Q), (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)NB * 8, (cuuint64_t)Q * NB * 8, (cuuint64_t)N * 8};
  cuuint32_t box[4] = {(cuuint32_t)C, 1, 256, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 4, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, tile_swizzle(C), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// first-pass output: column c's L outputs contiguous at c L + k: a (k % 16, c, k / 16, batch)
// view with strides (8, 8 L, 128, 8 N) bytes, box [16][C][L / 16][1], 128-byte swizzle
static bool map_out0(CUtensorMap* m, void* base, long long N, int L, int C, long long batch) {
  encode_fn enc = get_encode();
  if (!enc || L / 16 > 256) return false;
  cuuint64_t dims[4] = {16, (cuuint64_t)(N / L), (cuuint64_t)(L / 16), (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)L * 8, 128, (cuuint64_t)N * 8};
  cuuint32_t box[4] = {16, (cuuint32_t)C, (cuuint32_t)(L / 16), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// out (autosort write): a [batch][NB/Ns][L][Ns] view, box [C][min(L, 256)][1][1]
static bool map_out(CUtensorMap* m, void* base, long long N, int L, int C, long long Ns, long long batch) {
  encode_fn enc = get_encode();
  if (!enc) return false;
  const long long NB = N / L;
  cuuint64_t dims[4] = {(cuuint64_t)Ns, (cuuint64_t)L, (cuuint64_t)(NB / Ns), (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)Ns * 8, (cuuint64_t)Ns * L * 8, (cuuint64_t)N * 8};
  cuuint32_t box[4] = {(cuuint32_t)C, (cuuint32_t)(L < 256 ? L : 256), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             tile_swizzle(C), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool passes_available() { return get_encode() != nullptr; }

// Split N (power of two, 2^9 .. 2^48) into p passes: p = ceil(log2 N / 8) with lengths in
// [16, 256], except that 2^17 .. 2^20 take two passes of up to 1024, 2^21 .. 2^23 two passes
// with 2048/4096-long ones and 2^25 .. 2^28 three passes [<= 1024, <= 1024, 256] -- one HBM round
// trip fewer (measured on B200, profiles/r01h, r01j;
// env FFTC_PASS_MAXLOG=8 restores the short passes).  Lengths are
// as equal as possible, larger first.
int pass_split(long long N, int* Ls, int max) {
  if (N < 512 || (N & (N - 1))) return -1;
  int n = 0;
  while ((1LL << n) < N) ++n;
  int maxlog = 10;
  if (const char* m = getenv("FFTC_PASS_MAXLOG")) maxlog = atoi(m);
  if (maxlog < 8) maxlog = 8;
  if (maxlog > 10) maxlog = 10;
  if (const char* fl = getenv("FFTC_PASS_LOGS")) {  // tuning: explicit log2 lengths, e.g. "10,9,8"
    int q = 0, sum = 0;
    for (const char* c = fl; *c && q < max;) {
      const int e = atoi(c);
      if (e < 4 || e > 12) return -1;
      Ls[q++] = 1 << e;
      sum += e;
      while (*c && *c != ',') ++c;
      if (*c == ',') ++c;
    }
    if (sum == n) return q;
  }
  if (n >= 21 && n <= 23 && maxlog >= 10 && max >= 2) {
    // two passes with 2048/4096-long passes (2-column tiles first, 4-column tiles -- full 32-byte
    // sectors per strided row -- later): 2^21 [2048, 1024] 2.26 -> 1.69 ms, 2^22 [2048, 2048]
    // 2.20 -> 1.89 ms, 2^23 [4096, 2048] 2.22 -> 2.13 ms (profiles/r01j/long_first_pass.jsonl);
    // round 2, the register-resident 4096-long first pass (rpass.cu): 2^22 [4096, 1024] 1.78 ms,
    // 2^23 [4096, 2048] 1.93 ms (profiles/r02g)
    Ls[0] = n == 21 ? 2048 : 4096;
    Ls[1] = n == 21 ? 1024 : n == 22 ? 1024 : 2048;
    return 2;
  }
  int p = (n + 7) / 8;
  if (p == 3 && n <= 2 * maxlog) p = 2;  // 2^17 .. 2^20: two passes of <= 1024
  if (p == 4 && n <= 2 * maxlog + 8) {
    // 2^25 .. 2^28: three passes, the last one 256 long (16-column tiles: its autosort store
    // writes 128-byte rows; 8-column tiles there scatter 64-byte rows at MB strides, slower)
    if (max < 3) return -1;
    const int m = n - 8;
    Ls[0] = 1 << ((m + 1) / 2);
    Ls[1] = 1 << (m / 2);
    Ls[2] = 256;
    return 3;
  }
  if (p > max) return -1;
  for (int s = 0; s < p; ++s) {
    const int e = n / p + (s < n % p ? 1 : 0);
    if (e < 4 || e > maxlog) return -1;
    Ls[s] = 1 << e;
  }
  return p;
}

// Tiles per CTA group for pass length L of an N-point plan (adjacent column tiles back to back
// on one CTA: their strided TMA rows share 2 MB pages and DRAM rows).  Measured on B200
// (profiles/r01j/tile_groups.jsonl): 256-long and shorter passes 2 up to 2^20, 4 above (2^16
// 1.58 -> 1.44 ms, 2^24 2.40 -> 2.20 ms, 2^30 14.39 -> 13.13 ms); 512-long and longer passes
// 2, 3 from 2^28 (2^18 1.60 -> 1.51 ms, 2^28 2.62 -> 2.57 ms; 3 is slower for 2^25..2^27).
// Env FFTC_PASS_GROUP / FFTC_PASS_GROUP_LONG override (tuning), read at plan creation.
int pass_group(int L, long long N) {
  int grp = L >= 512 ? (N >= (1LL << 28) ? 3 : 2) : (N > (1LL << 20) ? 4 : 2);
  if (const char* gs = getenv(L >= 512 ? "FFTC_PASS_GROUP_LONG" : "FFTC_PASS_GROUP"))
    grp = atoi(gs) > 0 ? atoi(gs) : 1;
  return grp;
}

cudaError_t passes_execute(const PassPlanData& pp, const float2* in, float2* out, float2* work, long long batch,
                           int conj, cudaStream_t st) {
  // ping-pong so the last pass lands in `out`: pass s writes out if (p-1-s) even, else work
  const int p = pp.p;
  long long Ns = 1;
  const float2* src = in;
  for (int s = 0; s < p; ++s) {
    float2* dst = ((p - 1 - s) % 2 == 0) ? out : work;
    const PassEntry* e = pp.e[s];
    const int L = e->L;
    CUtensorMap tin, tout;
    if (e->cluster) {  // loads of one row residue class per CTA; outputs stored by the threads
      if (!map_in_cluster(&tin, src, pp.N, L, e->cols, e->cluster, batch)) return cudaErrorInvalidValue;
      tout = tin;
    } else {
      if (!map_in(&tin, src, pp.N, L, e->cols, batch)) return cudaErrorInvalidValue;
      if (s > 0 && !map_out(&tout, dst, pp.N, L, e->cols, Ns, batch)) return cudaErrorInvalidValue;
      if (s == 0 && !map_out0(&tout, dst, pp.N, L, e->cols, batch)) return cudaErrorInvalidValue;
    }
    PassGeom g{};
    g.tiles_per_batch = (int)(pp.N / L / e->cols);
    g.tiles_total = batch * g.tiles_per_batch;
    g.group = pp.group[s] > 0 ? pp.group[s] : 1;
    g.Ns = (int)Ns;
    g.N = pp.N;
    g.tw = s > 0;
    g.tws = pp.tws[s];
    cudaError_t err = e->launch(s == 0, tin, tout, dst, pp.tw[s], pp.twA[s], pp.twB[s], g, conj && s == 0,
                                conj && s == p - 1, st);
    if (err != cudaSuccess) return err;
    src = dst;
    Ns *= L;
  }
  return cudaSuccess;
}

}  // namespace fftc
