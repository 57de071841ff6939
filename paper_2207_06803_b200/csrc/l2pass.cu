// l2pass.cu -- L2-resident multi-pass path for large power-of-two N (product path).
//
// The multi-pass path (passes.cu) applies the paper's Eq. 2 at the pass
// level: N = L_0 L_1 ... L_{p-1}, each pass one Stockham level over the whole transform
// (passtile.cuh).  Run pass after pass over the whole batch, every element crosses HBM
// p times.  Here the batch is cut into chunks of tc whole transforms (~8 MiB) and every
// pass of a chunk runs while the chunk's intermediates are still in the 126 MB L2: pass 0
// reads the input from HBM, passes 1..p-2 read and write a ring of chunk-sized buffers
// that is re-used in place (so its lines stay dirty in L2 and are never written back),
// and pass p-1 writes the output to HBM.  Each element crosses HBM once (16 B), the
// single-pass minimum.
//
// One persistent (cooperative) kernel runs all passes of all chunks.  Work items are
// (chunk c, pass s, tile of 16 columns), numbered by ticket and dealt round-robin to the
// CTAs.  Tickets are ordered by phase k = c + lag s (within a phase, pass 0 first), so an
// item's inputs (pass s-1 of chunk c, phase k - lag) and the release of the ring slot it
// overwrites (phase k - 1 or earlier) are always earlier tickets: with every CTA resident
// the lowest unfinished ticket can always run, so dependency waits never deadlock.  Completion is tracked per (c, s) by two counters, tiles written (release
// after the stores are performed) and tiles read (release after the TMA load lands).
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include "l2pass.h"
#include "launch_util.h"
#include "passtile.cuh"

namespace fftc {

namespace {

struct Item {
  int c, s, tile, valid;
};

// q.ps[s] without a dynamic index into the parameter space (which would copy it to the stack)
__device__ __forceinline__ L2Stage stage_of(const L2Params& q, int s) {
  return s == 0 ? q.ps[0] : (s == 1 ? q.ps[1] : q.ps[2]);
}
__device__ __forceinline__ int tiles_of(const L2Params& q, int s) {
  return s == 0 ? q.ps[0].T : (s == 1 ? q.ps[1].T : q.ps[2].T);
}
__device__ __forceinline__ long long l2_ntrans(const L2Params& q, int c) {
  const long long r = q.B - (long long)c * q.tc;
  return r < q.tc ? r : q.tc;
}
// first ticket of phase k
__device__ __forceinline__ long long phase_start(const L2Params& q, long long k) {
  long long t = 0;
  for (int s = 0; s < q.p; ++s) {
    long long x = (k - (long long)q.lag * s) * q.tc;
    x = x < 0 ? 0 : (x > q.B ? q.B : x);
    t += x * tiles_of(q, s);
  }
  return t;
}
__device__ Item decode(const L2Params& q, long long x) {
  Item it{0, 0, 0, 0};
  const long long K = q.nchunks + (long long)q.lag * (q.p - 1);  // phases
  if (x >= phase_start(q, K)) return it;
  long long lo = 0, hi = K - 1;  // largest k with start(k) <= x
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (phase_start(q, mid) <= x) lo = mid;
    else hi = mid - 1;
  }
  long long off = x - phase_start(q, lo);
  for (int s = 0; s < q.p; ++s) {
    const long long c = lo - (long long)q.lag * s;
    if (c < 0 || c >= q.nchunks) continue;
    const long long sz = l2_ntrans(q, (int)c) * tiles_of(q, s);
    if (off < sz) {
      it.c = (int)c;
      it.s = s;
      it.tile = (int)off;
      it.valid = 1;
      return it;
    }
    off -= sz;
  }
  return it;
}
__device__ __forceinline__ unsigned* wdone(const L2Params& q, int c, int s) { return q.ctr + 1 + c * q.p + s; }
__device__ __forceinline__ unsigned* rdone(const L2Params& q, int c, int s) {
  return q.ctr + 1 + (q.nchunks + c) * q.p + s;
}
__device__ __forceinline__ int ring_slot(const L2Params& q, int c, int s) {
  return (int)(((long long)c * (q.p - 1) + s) % q.slots);
}
// The schedules' in-tile barriers as a named barrier over the 256 compute threads
// (the producer warp never joins them).
template <class Base>
struct Compute256 : Base {
  __device__ __forceinline__ static void sync() { named_sync1<256>(); }
};

constexpr int kStages = 3;          // shared-memory tile buffers per CTA
constexpr int kThreads = 256 + 32;  // 16 x 16 compute threads + one producer warp

// Warp-specialised persistent kernel.  Warp 8 (producer, one lane) takes tickets, waits
// for each item's dependencies and issues its TMA load into a free buffer (full/empty
// mbarrier pairs); warps 0-7 compute the pass tile and store it.  The compute side never
// waits on global memory: completion signals of a tile (fence + release) are issued after
// the next tile's compute, or at once when the compute side would otherwise block.
template <class PA, class PB, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_l2(const __grid_constant__ L2Params q) {
  static_assert(PA::THREADS == 256 && PB::THREADS == 256, "both schedules: 16 columns x 16 threads");
  using CA = Compute256<PA>;
  using CB = Compute256<PB>;
  constexpr int C = 16;
  constexpr int LMAX = PA::N;
  extern __shared__ __align__(1024) unsigned char smraw[];
  float2* buf0 = reinterpret_cast<float2*>(smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ Item s_item[kStages];
  if (threadIdx.x == 0) {
    for (int k = 0; k < kStages; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], 1);
    }
  }
  __syncthreads();

  if (threadIdx.x >= 256) {
    // ------------------------------------------------------------ producer
    // Static round-robin: this CTA runs tickets blockIdx.x, + gridDim.x, ...  (the launch is
    // cooperative, so every CTA is resident and the lowest unfinished ticket can always run).
    if (threadIdx.x != 256) return;
    const uint64_t pol_first = policy_evict_first();
    const uint64_t pol_last = policy_evict_last();
    const long long total = phase_start(q, q.nchunks + (long long)q.lag * (q.p - 1));
    int okw_c = -1, okw_s = -1, okr_c = -1, okr_s = -1;  // last counters seen complete
    int n = 0;
    for (long long x = blockIdx.x;; x += gridDim.x, ++n) {
      const int k = n % kStages;
      if (n >= kStages) mbar_wait(&empty[k], ((n / kStages) - 1) & 1);  // consumers released buffer k
      const Item it = x < total ? decode(q, x) : Item{0, 0, 0, 0};
      s_item[k] = it;
      if (!it.valid) {
        mbar_arrive(&full[k]);  // no transaction: consumers see the end marker
        return;
      }
      // inputs written (pass s-1 of chunk c complete)
      if (it.s > 0 && !(okw_c == it.c && okw_s == it.s - 1)) {
        const unsigned need = (unsigned)(l2_ntrans(q, it.c) * tiles_of(q, it.s - 1));
        while (ld_acquire_gpu(wdone(q, it.c, it.s - 1)) < need) __nanosleep(128);
        okw_c = it.c;
        okw_s = it.s - 1;
      }
      // output ring slot released by the reader of its previous occupant
      if (it.s < q.p - 1) {
        const long long prev = (long long)it.c * (q.p - 1) + it.s - q.slots;
        if (prev >= 0) {
          const int c2 = (int)(prev / (q.p - 1)), s2 = (int)(prev % (q.p - 1)) + 1;
          if (!(okr_c == c2 && okr_s == s2)) {
            const unsigned need = (unsigned)(l2_ntrans(q, c2) * tiles_of(q, s2));
            while (ld_acquire_gpu(rdone(q, c2, s2)) < need) __nanosleep(128);
            okr_c = c2;
            okr_s = s2;
          }
        }
      }
      const L2Stage ps = stage_of(q, it.s);
      const int t = it.tile / ps.T, c0 = (it.tile % ps.T) * C;
      fence_proxy_async_global();  // acquired generic-proxy writes before the async-proxy read
      mbar_arrive_expect_tx(&full[k], (uint32_t)ps.L * C * 8u);
      if (it.s == 0)
        tma_load_3d_hint(buf0 + k * LMAX * C, &q.ld[0], c0, 0, (int)((long long)it.c * q.tc + t), &full[k],
                         pol_first);
      else
        tma_load_3d_hint(buf0 + k * LMAX * C, &q.ld[it.s], c0, 0, ring_slot(q, it.c, it.s - 1) * q.tc + t,
                         &full[k], pol_last);
    }
  }

  // -------------------------------------------------------------- compute (threads 0..255)
  int f, lt;
  PA::thread_coords(threadIdx.x, f, lt);  // F_FAST, FPB 16: f = tid % 16, lt = tid / 16
  const uint64_t pol_first = policy_evict_first();
  const uint64_t pol_last = policy_evict_last();
  // thread 0's pending completion of the previous tile: buffer to release, counter to bump
  int pend_buf = -1, pend_kind = 0;  // kind 1: generic stores, 2: bulk store (+ counter), 3: bulk store only
  unsigned* pend_ctr = nullptr;
  auto flush = [&]() {
    if (pend_buf < 0) return;
    if (pend_kind == 1) {
      __threadfence();
      fence_proxy_async_global();
      red_release_gpu_add(pend_ctr, 1u);
    } else if (pend_kind == 2) {
      bulk_wait0();
      fence_proxy_async_global();
      red_release_gpu_add(pend_ctr, 1u);
    } else {
      bulk_wait_read0();
    }
    mbar_arrive(&empty[pend_buf]);
    pend_buf = -1;
  };
  for (int n = 0;; ++n) {
    const int k = n % kStages;
    const uint32_t ph = (n / kStages) & 1;
    if (threadIdx.x == 0 && !mbar_test(&full[k], ph)) flush();  // about to block: signal first
    mbar_wait(&full[k], ph);
    const Item it = s_item[k];
    if (!it.valid) break;
    const L2Stage ps = stage_of(q, it.s);
    float2* sm = buf0 + k * LMAX * C;
    const int t = it.tile / ps.T, c0 = (it.tile % ps.T) * C;
    if (threadIdx.x == 0 && it.s > 0) red_release_gpu_add(rdone(q, it.c, it.s), 1u);  // input slot read
    const float ci = it.s == 0 ? q.csign : 1.f, co = it.s == q.p - 1 ? q.csign : 1.f;
    if (it.s == 0) {  // pass 0 always runs the long schedule (lengths are non-increasing)
      pass_tile<CA, false>(sm, f, lt, c0 + f, 1, ps.tw, ps.twA, ps.twB, ps.tws, ci, co);
    } else if (ps.which == 0) {
      pass_tile<CA, true>(sm, f, lt, c0 + f, ps.Ns, ps.tw, ps.twA, ps.twB, ps.tws, ci, co);
    } else {
      pass_tile<CB, true>(sm, f, lt, c0 + f, ps.Ns, ps.tw, ps.twA, ps.twB, ps.tws, ci, co);
    }
    if (threadIdx.x == 0) flush();  // the previous tile's stores had a whole tile of compute to land
    if (it.s == 0) {
      // pass 0 -> ring slot: column c's outputs contiguous at c L + r
      named_sync1<256>();
      float2* go = q.ring + ((long long)ring_slot(q, it.c, 0) * q.tc + t) * q.N + (long long)c0 * ps.L;
      auto st = [&](float2* a, float2 v) { st_evict_last(a, v, pol_last); };
      pass0_store<CA>(sm, go, st);
      fence_proxy_async_smem();  // generic reads of the buffer before the next TMA write into it
      named_sync1<256>();
      if (threadIdx.x == 0) {
        pend_buf = k;
        pend_kind = 1;
        pend_ctr = wdone(q, it.c, 0);
      }
    } else {
      // autosort store of the [L][16] box: ring slot (middle pass) or the output (last pass)
      fence_proxy_async_smem();
      named_sync1<256>();
      if (threadIdx.x == 0) {
        const bool last = it.s == q.p - 1;
        const int b = last ? (int)((long long)it.c * q.tc + t) : ring_slot(q, it.c, it.s) * q.tc + t;
        tma_store_4d_hint(&q.st[it.s], sm, c0 % ps.Ns, 0, c0 / ps.Ns, b, last ? pol_first : pol_last);
        bulk_commit();
        pend_buf = k;
        pend_kind = last ? 3 : 2;
        pend_ctr = last ? nullptr : wdone(q, it.c, it.s);
      }
    }
  }
  if (threadIdx.x == 0) {
    flush();
    bulk_wait0();
  }
}

template <class PA, class PB, int MINB>
cudaError_t launch_l2(const L2Params& q, cudaStream_t st) {
  constexpr size_t smem = (size_t)kStages * PA::N * 16 * sizeof(float2) + 1024;
  auto kern = k_l2<PA, PB, MINB>;
  static PerDevice<KernelSetup> ks_pd;
  const KernelSetup& ks = ks_pd.get([&] { return kernel_setup(kern, kThreads, smem); });
  if (ks.err != cudaSuccess) return ks.err;
  const int grid_max = ks.grid_max;
  const char* g = getenv("FFTC_L2_GRID");  // tuning
  int grid = g ? atoi(g) : grid_max;
  if (grid > grid_max || grid < 1) grid = grid_max;
  // cooperative: all CTAs co-resident (the static ticket schedule relies on it)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, q);
}

}  // namespace

// the same radices as the HBM multi-pass kernels (passes.cu): both paths compute bit-identical results
using L2_256 = Sched<256, Radices<16, 16>, 16, 16, F_FAST, 0, LAY_TMA128>;
using L2_128 = Sched<128, Radices<16, 8>, 16, 16, F_FAST, 0, LAY_TMA128>;
using L2_64 = Sched<64, Radices<8, 8>, 16, 16, F_FAST, 0, LAY_TMA128>;
using L2_32 = Sched<32, Radices<8, 4>, 16, 16, F_FAST, 0, LAY_TMA128>;

// First entry per (LA, LB) = default; FFTC_L2_KERNEL=<name> pins a candidate (tuning).
static const L2Entry kL2[] = {
    {256, 256, &launch_l2<L2_256, L2_256, 2>, "l2_256x256_b2"},
    {256, 256, &launch_l2<L2_256, L2_256, 3>, "l2_256x256_b3"},
    {256, 128, &launch_l2<L2_256, L2_128, 2>, "l2_256x128_b2"},
    {256, 128, &launch_l2<L2_256, L2_128, 3>, "l2_256x128_b3"},
    {128, 128, &launch_l2<L2_128, L2_128, 2>, "l2_128x128_b2"},
    {128, 128, &launch_l2<L2_128, L2_128, 3>, "l2_128x128_b3"},
    {128, 64, &launch_l2<L2_128, L2_64, 2>, "l2_128x64_b2"},
    {128, 64, &launch_l2<L2_128, L2_64, 3>, "l2_128x64_b3"},
    {64, 64, &launch_l2<L2_64, L2_64, 3>, "l2_64x64_b3"},
    {64, 32, &launch_l2<L2_64, L2_32, 3>, "l2_64x32_b3"},
};

int l2_split(long long N, int* Ls, int max) {
  if (N < 8192 || (N & (N - 1))) return -1;
  int n = 0;
  while ((1LL << n) < N) ++n;
  if (n > 21) return -1;
  const int p = n <= 16 ? 2 : 3;
  if (p > max) return -1;
  for (int s = 0; s < p; ++s) {
    const int e = n / p + (s < n % p ? 1 : 0);
    if (e < 5 || e > 8) return -1;
    Ls[s] = 1 << e;
  }
  return p;
}

const L2Entry* find_l2(const int* Ls, int p) {
  int a = Ls[0], b = Ls[0];
  for (int s = 1; s < p; ++s) {
    a = Ls[s] > a ? Ls[s] : a;
    b = Ls[s] < b ? Ls[s] : b;
  }
  if (const char* want = getenv("FFTC_L2_KERNEL"))
    for (const auto& e : kL2)
      if (e.LA == a && e.LB == b && strcmp(e.name, want) == 0) return &e;
  for (const auto& e : kL2)
    if (e.LA == a && e.LB == b) return &e;
  return nullptr;
}

void l2_geometry(long long N, long long batch, int p, int* tc, int* slots, int* lag) {
  long long chunk = 8LL << 20;
  if (const char* m = getenv("FFTC_L2_CHUNK_MB")) chunk = atoll(m) << 20;
  long long t = chunk / (N * 8);
  if (t < 1) t = 1;
  long long pw = 1;
  while (pw * 2 <= t) pw *= 2;
  if (batch > 0 && pw > batch) pw = batch;
  *tc = (int)pw;
  int g = 2;
  if (const char* m = getenv("FFTC_L2_LAG")) g = atoi(m);
  if (g < 1) g = 1;
  *lag = g;
  // pass s of chunk c runs in phase c + lag s: its input was written lag phases earlier, and the
  // ring slot it overwrites was last read lag + 1 phases earlier (see the producer)
  *slots = (p - 1) * (g + 2);
}

static long long nchunks_of(const L2PlanData& d, long long batch) { return (batch + d.tc - 1) / d.tc; }

size_t l2_work_bytes(const L2PlanData& d, long long batch) {
  const size_t ring = (size_t)d.slots * d.tc * d.N * sizeof(float2);
  const size_t ctr = (size_t)(1 + 2 * nchunks_of(d, batch) * d.p) * sizeof(unsigned);
  return ring + ((ctr + 255) & ~(size_t)255);
}

// ---------------------------------------------------------------- host: tensor maps
typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static encode_fn get_encode() {
  static encode_fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = (encode_fn)p;
  }
  return fn;
}
// a [batch][L rows][N/L cols] view, box [16 cols][L rows][1]
static bool map_cols(CUtensorMap* m, const void* base, long long N, int L, long long batch) {
  const long long NB = N / L;
  cuuint64_t dims[3] = {(cuuint64_t)NB, (cuuint64_t)L, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)NB * 8, (cuuint64_t)N * 8};
  cuuint32_t box[3] = {16, (cuuint32_t)L, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, const_cast<void*>(base), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// the autosort write of a pass: a [batch][NB/Ns][L][Ns] view, box [16][L][1][1]
static bool map_autosort(CUtensorMap* m, void* base, long long N, int L, long long Ns, long long batch) {
  const long long NB = N / L;
  cuuint64_t dims[4] = {(cuuint64_t)Ns, (cuuint64_t)L, (cuuint64_t)(NB / Ns), (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)Ns * 8, (cuuint64_t)Ns * L * 8, (cuuint64_t)N * 8};
  cuuint32_t box[4] = {16, (cuuint32_t)L, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 4, base, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t l2_execute(const L2PlanData& d, const float2* in, float2* out, void* work, long long batch, int conj,
                       cudaStream_t st) {
  if (batch == 0) return cudaSuccess;
  if (!get_encode()) return cudaErrorNotSupported;
  L2Params q;
  memset(&q, 0, sizeof(q));
  q.N = d.N;
  q.B = batch;
  q.p = d.p;
  q.tc = d.tc;
  q.nchunks = (int)nchunks_of(d, batch);
  q.slots = d.slots;
  q.lag = d.lag;
  q.csign = conj ? -1.f : 1.f;
  q.ring = reinterpret_cast<float2*>(work);
  q.ctr = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(work) + (size_t)d.slots * d.tc * d.N * sizeof(float2));
  const long long ring_b = (long long)d.slots * d.tc;
  long long Ns = 1;
  for (int s = 0; s < d.p; ++s) {
    L2Stage& ps = q.ps[s];
    ps.L = d.L[s];
    ps.which = d.L[s] == d.e->LA ? 0 : 1;
    ps.Ns = (int)Ns;
    ps.T = (int)(d.N / d.L[s] / 16);
    ps.tw = d.tw[s];
    ps.twA = d.twA[s];
    ps.twB = d.twB[s];
    ps.tws = d.tws[s];
    bool ok = s == 0 ? map_cols(&q.ld[0], in, d.N, d.L[0], batch) : map_cols(&q.ld[s], q.ring, d.N, d.L[s], ring_b);
    if (ok && s > 0)
      ok = s == d.p - 1 ? map_autosort(&q.st[s], out, d.N, d.L[s], Ns, batch)
                        : map_autosort(&q.st[s], q.ring, d.N, d.L[s], Ns, ring_b);
    if (!ok) return cudaErrorInvalidValue;
    Ns *= d.L[s];
  }
  cudaError_t e = cudaMemsetAsync(q.ctr, 0, (size_t)(1 + 2 * q.nchunks * q.p) * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  return d.e->launch(q, st);
}

}  // namespace fftc
