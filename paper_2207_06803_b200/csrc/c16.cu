// c16.cu -- N = 65536 in ONE HBM round trip on a cluster of eight CTAs (product path).
//
// The paper's Eq. 2 once at the top with M = K = 256 (the four-step of DESIGN §5):
// view x as A[q][r] = x[256 q + r]; DFT_256 down every column r -> Y[j][r]; multiply by w_N^{r j};
// DFT_256 along every row j -> Z[j][k1]; X[j + 256 k1] = Z[j][k1].  Both DFT_256 are Eq. 2 again
// (two radix-16 Stockham stages, fused.cuh header).  A transform is 512 KB, so it is spread over
// a cluster of 8 CTAs (one per SM, 64 KB each; 16 CTAs at two per SM as an option): CTA p loads
// columns [32 p, 32 p + 32) of A (one TMA box, 256-byte rows), transforms them, and stores element
// (j, r) of Y straight into the shared memory of CTA j div 32 (distributed shared memory), which
// then owns rows [32 p', 32 p' + 32) for the row DFTs and writes X[j + 256 k1] for its rows.
// HBM sees 8 + 8 bytes per element (the single-pass minimum) instead of the 32 of two passes.
//
// The twiddle w_N^{r j} is folded into the row DFT: with r = i + 16 s (stage B1 butterfly i, input
// s) and the deferred factor u^i (u = w_N^j) landing on stage B2's input slot s2 = i, stage B1
// multiplies input s by w_N^{16 j s} and stage B2 input s2 by w_N^{(256 i2 + j) s2} (= (w_256^{i2}
// u)^{s2}, replacing the stage twiddle) -- no separate twiddle pass.  Powers 1, 2, 4, 8 come from
// the two-level table and the rest as single products of those: a power tree grown from one value
// multiplies its phase error by the exponent (2.7e-6 rel-L2 measured with u^16 by squaring).
//
// 512 threads per CTA, one radix-16 butterfly each per stage.  Rows travel as st.async remote
// stores counted on the receiver's mbarrier (complete_tx, 64 KB per transform), so no release
// fence waits for the global stores (a release cluster barrier compiled to MEMBAR.ALL.GPU and a
// first version stalled on it).  A sender delivers into B[x] only after every receiver has
// arrived (remotely, CTA-scope release) on the sender's bfree[x] mbarrier -- no cluster barrier in
// the loop, whose acquire wait also invalidated L1 (CCTL.IVALL) and with it the twiddle tables.
// Measured on B200 (profiles/r02g): 1.73-1.79 ms per 2^28 elements against 1.45 ms for the two
// 256-long passes -- instruction-bound (87 thread instructions per element, 45 % issue) on the
// 120 SMs that 15 resident clusters of 8 occupy; staging the rows in shared memory and sending
// eight 8 KB bulk copies instead of st.async ran at the same speed.
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include "c16.h"
#include "launch_util.h"
#include "passtile.cuh"
#include "tma.cuh"

namespace fftc {

namespace {

constexpr int kN = 65536, kS = 256, kR = 16;
constexpr int kCPitch = 257;  // B rows in the row phase (odd pitch)

// asynchronous 8-byte store into another CTA's shared memory, counted on that CTA's mbarrier
// (complete_tx): no release fence -- the receiver's mbarrier wait makes the data visible
__device__ __forceinline__ void st_async_f2(uint32_t addr, float2 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "f"(v.x), "f"(v.y), "r"(bar)
               : "memory");
}
// XOR swizzle of a row-phase column index: low 4 bits ^= bits 4..7
__device__ __forceinline__ int swz(int c) { return c ^ ((c >> 4) & 15); }

// w[r] = w_N^{e r} for r = 1..15: r = 1, 2, 4, 8 from the two-level table (A[t] = w_N^t, t < 256;
// B[h] = w_N^{256 h}), the others as products of two of those (as the stage tables are used)
__device__ __forceinline__ void root_powers(const float2* __restrict__ twA, const float2* __restrict__ twB, int e,
                                            float2 (&w)[kR]) {
  sfor<kR - 1>([&](auto r_) {
    constexpr int r = decltype(r_)::value + 1;
    constexpr int hb = highbit(r);
    if constexpr (hb == r) {
      const int x = (e * r) & (kN - 1);
      w[r] = cmul(__ldg(twA + (x & 255)), __ldg(twB + (x >> 8)));
    } else {
      w[r] = cmul(w[hb], w[r - hb]);
    }
  });
}
// w_256^{m s} for s = 1..15 from the plan's DFT_256 stage table (stage 1 entries (16 - 1) + (s - 1) 16 + m)
__device__ __forceinline__ void stage_tw(const float2* __restrict__ tw, int m, float2 (&w)[kR]) {
  const float2* t = tw + 15 + m;
  sfor<kR - 1>([&](auto r_) {
    constexpr int r = decltype(r_)::value + 1;
    constexpr int hb = highbit(r);
    if constexpr (hb == r) w[r] = __ldg(t + (r - 1) * 16);
    else w[r] = cmul(w[hb], w[r - hb]);
  });
}

// Software pipeline over the cluster's transforms: iteration t runs the column phase of t (its
// rows leave by st.async as soon as they are computed) and then the row phase of t - 1, whose
// rows arrived during the column phase -- the DSMEM delivery overlaps arithmetic instead of
// being waited for.  Shared memory: A (the TMA tile; the column-phase stage exchange in place),
// B[2] (incoming rows of two transforms, [rows][257]; the row-phase exchange in place).  Flow
// control per buffer x: bfull[x] (the receiver's 64 KB of rows, complete_tx) and bfree[x] (the
// sender may deliver transform t into B[x] once all receivers arrived after consuming t - 2).
// Q CTAs per cluster (launched with a runtime cluster dimension): CTA p owns kCols = 256 / Q
// columns in the column phase and as many rows in the row phase, with 16 kCols threads (one
// radix-16 butterfly each per stage).  Q = 8: 64 KB per CTA and transform, one CTA per SM (512
// threads, 194 KB of shared memory); Q = 16: 32 KB, 256 threads, two CTAs per SM.
template <int Q>
__global__ void __launch_bounds__(16 * (kS / Q), Q / 8)
    k_c16(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out, const float2* __restrict__ tw,
          const float2* __restrict__ twA, const float2* __restrict__ twB, long long batch, float csign_in,
          float csign_out) {
  constexpr int kQ = Q, kCols = kS / Q;
  constexpr uint32_t kTileBytes = (uint32_t)kS * kCols * 8u;  // per CTA and transform
  extern __shared__ unsigned char smraw[];
  float2* A = reinterpret_cast<float2*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
  float2* Bbuf = A + kS * kCols;  // two [kCols][kCPitch] buffers
  __shared__ __align__(8) uint64_t full, bfull[2], bfree[2];
  const int p = (int)cluster_ctarank();
  const long long cid = blockIdx.x / kQ, ncl = gridDim.x / kQ;
  const int t = (int)threadIdx.x;
  auto issue = [&](long long b) {
    mbar_arrive_expect_tx(&full, kTileBytes);
    tma_load_3d(A, &tin, p * kCols, 0, (int)b, &full);
  };
  if (t == 0) {
    mbar_init(&full, 1);
    mbar_init(&bfull[0], 1);
    mbar_init(&bfull[1], 1);
    mbar_init(&bfree[0], kQ);  // one arrive from every receiver once it has consumed B[x]
    mbar_init(&bfree[1], kQ);
    fence_mbarrier_init_cluster();
  }
  cluster_sync_all();  // every CTA's barriers exist before a peer signals them
  if (t == 0 && cid < batch) issue(cid);
  const uint32_t B_local = smem_u32(Bbuf), bfull_local = smem_u32(&bfull[0]), bfree_local = smem_u32(&bfree[0]);
  const long long nt = cid < batch ? (batch - 1 - cid) / ncl + 1 : 0;  // this cluster's transforms
  // row phase of the cluster's transform `it` (rows in B[it & 1])
  auto row_phase = [&](long long it) {
    float2 v[kR];
    float2* B = Bbuf + (it & 1) * (kCols * kCPitch);
    const long long b = cid + it * ncl;
    mbar_wait(&bfull[it & 1], (uint32_t)((it >> 1) & 1));
    {  // B1 thread (i, jl): butterfly i of row jl; input s times w_N^{16 j s}
      const int i = t % 16, jl = t / 16;
      const int j = p * kCols + jl;
      sfor<kR>([&](auto s_) {
        constexpr int s = decltype(s_)::value;
        v[s] = B[jl * kCPitch + i + 16 * s];
      });
      float2 w[kR];
      root_powers(twA, twB, 16 * j, w);
      sfor<kR - 1>([&](auto s_) {
        constexpr int s = decltype(s_)::value + 1;
        v[s] = cmul(v[s], w[s]);
      });
      Codelet<kR>::run(v);  // B1 (Ns = 1): outputs at 16 i + s'
      __syncthreads();      // every B1 read precedes the in-place writes
      sfor<kR>([&](auto s_) {
        constexpr int s = decltype(s_)::value;
        B[jl * kCPitch + swz(16 * i + s)] = v[s];
      });
    }
    __syncthreads();
    {  // B2 thread (jl, i2): input s2 times w_N^{(256 i2 + j) s2}; outputs k1 = i2 + 16 s''
      const int jl = t % kCols, i2 = t / kCols;
      const int j = p * kCols + jl;
      sfor<kR>([&](auto s_) {
        constexpr int s = decltype(s_)::value;
        v[s] = B[jl * kCPitch + swz(i2 + 16 * s)];
      });
      float2 w[kR];
      root_powers(twA, twB, 256 * i2 + j, w);
      sfor<kR - 1>([&](auto s_) {
        constexpr int s = decltype(s_)::value + 1;
        v[s] = cmul(v[s], w[s]);
      });
      // B[it & 1] consumed (every loaded value used above): expect transform it + 2's rows in it
      if (it + 2 < nt) {  // B[it & 1] will receive transform it + 2
        if (t == 0) mbar_arrive_expect_tx(&bfull[it & 1], kTileBytes);
        fence_proxy_async_smem();  // generic reads of B before the peers' asynchronous stores into it
        __syncthreads();           // every thread has consumed B[it & 1]
        // tell every sender (release at CTA scope orders this CTA's reads before its stores)
        if (t < kQ) mbar_arrive_remote(dsmem_map(bfree_local + (uint32_t)((it & 1) * 8), (uint32_t)t));
      }
      Codelet<kR>::run(v);
      float2* o = out + b * kN + j + kS * i2;
      sfor<kR>([&](auto s_) {
        constexpr int s = decltype(s_)::value;
        __stcs(o + kS * 16 * s, make_float2(v[s].x, csign_out * v[s].y));
      });
    }
  };
  if (t == 0) {
    if (nt > 0) mbar_arrive_expect_tx(&bfull[0], kTileBytes);
    if (nt > 1) mbar_arrive_expect_tx(&bfull[1], kTileBytes);
  }
  for (long long it = 0; it < nt; ++it) {
    const long long b = cid + it * ncl;
    float2 v[kR];
    // ---- column phase: thread (rl, ja) = column 32 p + rl, butterfly ja of stages A1 and A2
    const int rl = t % kCols, ja = t / kCols;
    mbar_wait(&full, (uint32_t)(it & 1));
    sfor<kR>([&](auto s_) {
      constexpr int s = decltype(s_)::value;
      float2 x = A[(ja + 16 * s) * kCols + rl];
      x.y *= csign_in;
      v[s] = x;
    });
    Codelet<kR>::run(v);  // A1 (Ns = 1): outputs at 16 ja + s'
    __syncthreads();      // every A1 read precedes the in-place writes
    sfor<kR>([&](auto s_) {
      constexpr int s = decltype(s_)::value;
      A[(16 * ja + s) * kCols + rl] = v[s];
    });
    __syncthreads();
    sfor<kR>([&](auto s_) {
      constexpr int s = decltype(s_)::value;
      v[s] = A[(ja + 16 * s) * kCols + rl];
    });
    fence_proxy_async_smem();
    __syncthreads();  // A read: the next transform of this cluster may stream in
    if (t == 0 && it + 1 < nt) issue(b + ncl);
    {  // A2 (Ns = 16): twiddle w_256^{ja s}, outputs j = ja + 16 s''
      float2 w[kR];
      stage_tw(tw, ja, w);
      sfor<kR - 1>([&](auto s_) {
        constexpr int s = decltype(s_)::value + 1;
        v[s] = cmul(v[s], w[s]);
      });
      Codelet<kR>::run(v);
    }
    // ---- deliver Y[j][kCols p + rl] (j = ja + 16 s) to CTA j div kCols = 16 s div kCols, row
    // j mod kCols = 16 s mod kCols + ja, buffer it & 1
    // every CTA has consumed B[it & 1] (transform it - 2): the receivers' arrives on bfree
    if (it >= 2) mbar_wait(&bfree[it & 1], (uint32_t)(((it >> 1) - 1) & 1));
    const uint32_t boff = (uint32_t)((it & 1) * (kCols * kCPitch) + p * kCols + rl) * 8u;
    sfor<kR>([&](auto s_) {
      constexpr int s = decltype(s_)::value;
      constexpr int dst = 16 * s / kCols, row0 = 16 * s % kCols;
      st_async_f2(dsmem_map(B_local + boff + (uint32_t)((row0 + ja) * kCPitch * 8), dst), v[s],
                  dsmem_map(bfull_local + (uint32_t)((it & 1) * 8), dst));
    });
    // ---- row phase of the previous transform (its rows arrived during this column phase)
    if (it > 0) row_phase(it - 1);
  }
  if (nt > 0) row_phase(nt - 1);
  // nothing reaches this CTA's shared memory any more: every delivery into it completed before its
  // bfull waits, and the receivers' bfree arrives stop two transforms before the end
}

typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
encode_fn get_encode() {
  static encode_fn fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) == cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = (encode_fn)q;
  }
  return fn;
}

}  // namespace

bool c16_available() { return get_encode() != nullptr; }

template <int Q>
cudaError_t c16_launch(const CUtensorMap& tin, float2* out, long long batch, int conj, const float2* tw256,
                       const float2* twA, const float2* twB, cudaStream_t st) {
  constexpr int kCols = kS / Q, kThreads = 16 * kCols;
  constexpr size_t smem = (size_t)(kS * kCols + 2 * kCols * kCPitch) * sizeof(float2) + 128;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = Q;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  struct Setup {
    cudaError_t err;
    int clusters;
  };
  static PerDevice<Setup> setup_pd;
  const Setup& su = setup_pd.get([&] {
    Setup s{cudaFuncSetAttribute(k_c16<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), 0};
    if (s.err == cudaSuccess && Q > 8)
      s.err = cudaFuncSetAttribute(k_c16<Q>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t c = cfg;
    c.gridDim = dim3(Q, 1, 1);
    if (s.err == cudaSuccess) s.err = cudaOccupancyMaxActiveClusters(&s.clusters, k_c16<Q>, &c);
    if (s.err == cudaSuccess && s.clusters <= 0) s.err = cudaErrorNotSupported;
    return s;
  });
  if (su.err != cudaSuccess) return su.err;
  const long long ncl = batch < su.clusters ? batch : su.clusters;
  cfg.gridDim = dim3((unsigned)(ncl * Q), 1, 1);
  return cudaLaunchKernelEx(&cfg, k_c16<Q>, tin, out, tw256, twA, twB, batch, conj ? -1.f : 1.f,
                            conj ? -1.f : 1.f);
}

cudaError_t c16_execute(const float2* in, float2* out, long long batch, int conj, const float2* tw256,
                        const float2* twA, const float2* twB, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  encode_fn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  // cluster size 8 (one CTA per SM); FFTC_C16_Q=16: clusters of 16 with two CTAs per SM (measured
  // 1.82 vs 1.73-1.79 ms per 2^28 elements: only 14 clusters of 16 fit, 20 % warps active)
  const char* qs = getenv("FFTC_C16_Q");
  const int q = qs && atoi(qs) == 16 ? 16 : 8;
  // in as [batch][256 rows q][256 columns r], box [256 / Q columns][256 rows][1]
  CUtensorMap tin;
  cuuint64_t dims[3] = {(cuuint64_t)kS, (cuuint64_t)kS, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)kS * 8, (cuuint64_t)kN * 8};
  cuuint32_t box[3] = {(cuuint32_t)(kS / q), (cuuint32_t)kS, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc(&tin, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, const_cast<float2*>(in), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (q == 16) return c16_launch<16>(tin, out, batch, conj, tw256, twA, twB, st);
  return c16_launch<8>(tin, out, batch, conj, tw256, twA, twB, st);
}

}  // namespace fftc

