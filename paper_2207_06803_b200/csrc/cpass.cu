// cpass.cu -- a 4096-long Stockham pass on a cluster of four CTAs (product path).
//
// One level of the paper's Eq. 2 at the pass level with L = 4096 (passes.cu
// header), its DFT_4096 of every column split once more by Eq. 2 across the CTAs of a cluster:
// with the column's rows r = 4 i + q,
//   X[k' + 1024 s] = sum_q w_4096^{q k'} w_4^{q s} Y_q[k'],   Y_q = DFT_1024(x[4 i + q]),
// so CTA q of the cluster loads only rows = q (mod 4) of C = 8 adjacent columns (a 64 KB tile,
// TMA, 64-byte rows) and runs the 1024-point sub-DFT in its own shared memory (the same pass_tile
// as the 1024-long pass kernel, input twiddle w^{m (4 i + q)}).  Outputs k' in [256 p, 256 p + 256)
// belong to CTA p: rows [256 p, 256 p + 256) of every Y_q tile are one contiguous 16 KB chunk, which
// CTA q pushes into CTA p's receive slot q with a shared -> peer-shared bulk copy (completion on
// CTA p's mbarrier).  CTA p then forms its outputs from its own chunk and the three received ones
// and stores them to HBM.  No cluster barrier in the loop: a CTA that has consumed its receive
// slots arrives on the three senders' `ack` mbarriers, which frees both the senders' tile buffer
// (its chunks were delivered) and the receiver's slots for the next tile.  A 4096-long pass needs
// >= 64-byte rows to stream at HBM speed, i.e. 256 KB of tile: more than one SM holds, hence the
// cluster.
#include <cuda.h>

#include "launch_util.h"
#include "passes.h"
#include "passtile.cuh"
#include "tma.cuh"

namespace fftc {

namespace {

constexpr int kQ = 4;     // CTAs per cluster = residue classes of the rows
constexpr int kNBuf = 2;  // tile buffers per CTA (+ kQ receive slots of a quarter tile)

template <class P, bool FIRST>
__global__ void __cluster_dims__(kQ, 1, 1) __launch_bounds__(P::THREADS, 1)
    k_cpass(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out, const float2* __restrict__ tw,
            const float2* __restrict__ twA, const float2* __restrict__ twB, PassGeom g, float csign_in,
            float csign_out) {
  constexpr int L1 = P::N, C = P::FPB, L = kQ * L1, BOX = 256;
  static_assert(C == 8 && L1 == 1024, "8-column tiles of 1024 rows per CTA");
  constexpr uint32_t TILE_BYTES = (uint32_t)L1 * C * 8u;
  constexpr uint32_t CHUNK = TILE_BYTES / kQ;  // rows [256 p, 256 p + 256): contiguous in LAY_TMA64
  constexpr int CHUNK_F2 = (int)(CHUNK / 8u);
  extern __shared__ __align__(1024) unsigned char smraw[];
  float2* buf0 = reinterpret_cast<float2*>(smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));
  float2* recv = buf0 + kNBuf * L1 * C;  // slot p: sender p's chunk for this CTA (own slot unused)
  __shared__ __align__(8) uint64_t full[kNBuf];
  __shared__ __align__(8) uint64_t rfull, ack;
  const int q = (int)cluster_ctarank();
  const long long cid = blockIdx.x / kQ, ncl = gridDim.x / kQ;
  int f, lt;
  P::thread_coords(threadIdx.x, f, lt);
  const long long T = g.tiles_total;
  const int tpb = g.tiles_per_batch;
  auto issue = [&](long long t, int k) {
    const int b = (int)(t / tpb), c0 = (int)(t % tpb) * C;
    mbar_arrive_expect_tx(&full[k], TILE_BYTES);
    sfor<L1 / BOX>([&](auto h_) {
      constexpr int h = decltype(h_)::value;
      tma_load_4d(buf0 + k * L1 * C + h * BOX * C, &tin, c0, q, h * BOX, b, &full[k]);
    });
  };
  if (threadIdx.x == 0) {
    for (int k = 0; k < kNBuf; ++k) mbar_init(&full[k], 1);
    mbar_init(&rfull, 1);
    mbar_init(&ack, kQ - 1);
    fence_mbarrier_init_cluster();
  }
  cluster_sync_all();  // every CTA's barriers exist before any peer signals them
  // groups of g.group adjacent tiles per cluster (their strided rows share pages), dealt round-robin
  const int grp = g.group;
  auto tile_of = [&](int i) -> long long { return ((long long)(i / grp) * ncl + cid) * grp + (i % grp); };
  if (threadIdx.x == 0)
    for (int k = 0; k < kNBuf; ++k)
      if (tile_of(k) < T) issue(tile_of(k), k);
  const long long Ns = g.Ns;
  // combine mapping: lanes across the 8 columns (a 64-byte row of the tile, and adjacent autosort
  // positions / sector-complete runs of the contiguous first-pass outputs), 4 rows per warp
  const int ff = (int)threadIdx.x % C;
  const int k0 = (int)threadIdx.x / C;
  constexpr int KSTEP = P::THREADS / C;
  const uint32_t rfull_p[3] = {dsmem_map(smem_u32(&rfull), (q + 1) % kQ), dsmem_map(smem_u32(&rfull), (q + 2) % kQ),
                               dsmem_map(smem_u32(&rfull), (q + 3) % kQ)};
  for (int it = 0; tile_of(it) < T; ++it) {
    const long long t = tile_of(it);
    const int k = it % kNBuf;
    float2* sm = buf0 + k * L1 * C;
    const int b = (int)(t / tpb), c0 = (int)(t % tpb) * C;
    if (threadIdx.x == 0) mbar_arrive_expect_tx(&rfull, (kQ - 1) * CHUNK);
    mbar_wait(&full[k], (it / kNBuf) & 1);
    // Y_q = DFT_1024 of rows 4 i + q of columns c0 .. c0 + 7 (input twiddle w^{m (4 i + q)}), in place
    pass_tile<P, !FIRST>(sm, f, lt, c0 + f, g.Ns, tw, twA, twB, g.tws, csign_in, 1.0f, nullptr, kQ, q);
    fence_proxy_async_smem();  // the sub-DFT's shared writes before the bulk copies read them
    __syncthreads();
    if (threadIdx.x == 0) {
      // chunk p -> CTA p's receive slot q (its peers' slots are free: acknowledged last tile)
      sfor<kQ - 1>([&](auto j_) {
        constexpr int j = decltype(j_)::value + 1;
        const int p = (q + j) % kQ;
        bulk_s2peer(dsmem_map(smem_u32(recv + q * CHUNK_F2), p), sm + p * CHUNK_F2, CHUNK, rfull_p[j - 1]);
      });
    }
    mbar_wait(&rfull, it & 1);  // the three peers' chunks for this CTA's outputs have landed
    const long long cc = c0 + ff;
    float2* gs = out + (long long)b * g.N + (FIRST ? cc * L : (cc / Ns) * Ns * L + (cc % Ns));
    const long long step = FIRST ? 1 : Ns;  // output row k -> gs + k step
    const float2* cb[kQ];  // the four Y_p chunks of this CTA's outputs: own tile or receive slot
    sfor<kQ>([&](auto p_) {
      constexpr int p = decltype(p_)::value;
      cb[p] = p == q ? sm + q * CHUNK_F2 : recv + p * CHUNK_F2;
    });
    constexpr int U = (L1 / kQ) * C / P::THREADS;
    sfor<U>([&](auto u_) {
      constexpr int u = decltype(u_)::value;
      const int kr = k0 + KSTEP * u;  // row within the chunk
      const int kp = q * (L1 / kQ) + kr;
      const int pos = P::sidx(ff, kp) - q * CHUNK_F2;  // position within a chunk (same swizzle phase)
      float2 z[kQ];
      sfor<kQ>([&](auto p_) {
        constexpr int p = decltype(p_)::value;
        z[p] = cb[p][pos];
      });
      sfor<kQ - 1>([&](auto p_) {
        constexpr int p = decltype(p_)::value + 1;
        z[p] = cmul(z[p], root_lookup_s(twA, twB, (long long)(p * kp) * Ns, g.tws));
      });
      Codelet<kQ>::run(z);
      sfor<kQ>([&](auto s_) {
        constexpr int sidx_ = decltype(s_)::value;
        __stcs(gs + (long long)(kp + sidx_ * L1) * step, make_float2(z[sidx_].x, csign_out * z[sidx_].y));
      });
    });
    __syncthreads();  // this tile's receive slots and own chunk are consumed
    if (threadIdx.x == 0) {
      sfor<kQ - 1>([&](auto j_) {
        constexpr int j = decltype(j_)::value + 1;
        mbar_arrive_remote(dsmem_map(smem_u32(&ack), (q + j) % kQ));
      });
      // every peer consumed this CTA's chunks: the tile buffer is free, the peers' slots too
      mbar_wait(&ack, it & 1);
      if (tile_of(it + kNBuf) < T) {
        fence_proxy_async_smem();
        issue(tile_of(it + kNBuf), k);
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

template <class P>
cudaError_t launch_cpass(bool first, const CUtensorMap& tin, const CUtensorMap&, float2* out, const float2* tw,
                         const float2* twA, const float2* twB, const PassGeom& g, int conj_in, int conj_out,
                         cudaStream_t st) {
  constexpr size_t smem = (size_t)(kNBuf + 1) * P::N * P::FPB * sizeof(float2) + 1024;
  auto kern = first ? k_cpass<P, true> : k_cpass<P, false>;
  static PerDevice<int> grid_pd[2];
  const int gmax = grid_pd[first ? 1 : 0].get([&] {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kQ * 64);
    cfg.blockDim = dim3(P::THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = kQ;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return 0;
    return n * kQ;
  });
  if (gmax <= 0) return cudaErrorInvalidConfiguration;
  if (g.tiles_total == 0) return cudaSuccess;
  const long long groups = (g.tiles_total + g.group - 1) / g.group;
  const long long clusters = groups < gmax / kQ ? groups : gmax / kQ;
  kern<<<(unsigned)(clusters * kQ), P::THREADS, smem, st>>>(tin, out, tw, twA, twB, g, conj_in ? -1.f : 1.f,
                                                            conj_out ? -1.f : 1.f);
  return cudaGetLastError();
}

}  // namespace

using CPRad_32x32 = Radices<32, 32>;
// the sub-DFT schedule of the 1024-long pass kernel (8 columns, 64-byte TMA rows, 32 x 32).
// Measured alternative: 512 threads (64 per column, 16 x 16 x 4) -- 4.39 vs 4.14 ms for 2^24.
using CPSched = Sched<1024, CPRad_32x32, 32, 8, F_FAST, 0, LAY_TMA64>;

cudaError_t launch_cpass4096(bool first, const CUtensorMap& tin, const CUtensorMap& tout, float2* out,
                             const float2* tw, const float2* twA, const float2* twB, const PassGeom& g, int conj_in,
                             int conj_out, cudaStream_t st) {
  return launch_cpass<CPSched>(first, tin, tout, out, tw, twA, twB, g, conj_in, conj_out, st);
}

}  // namespace fftc
