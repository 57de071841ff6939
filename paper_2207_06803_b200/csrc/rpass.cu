// rpass.cu -- a 4096-long Stockham pass whose tile lives in registers (product path).
//
// One level of the paper's Eq. 2 at the pass level with L = 4096 (passes.cu
// header): column c < N/L reads a[c + r N/L], multiplies by w_{Ns L}^{(c mod Ns) r} (later
// passes), runs DFT_4096 = three radix-16 Stockham stages (each one level of Eq. 2 again, fused.cuh
// header), and writes b[(c div Ns) Ns L + (c mod Ns) + k Ns].
//
// Why a separate kernel.  A 4096-long pass needs >= 32-byte row segments per strided row (4
// columns: a 128 KB tile) -- with 2 columns the half-sector rows run at under half speed -- and the
// next tile's load in flight while the current one is computed.  The shared-memory pass kernels
// hold the tile being computed in shared memory, so a 4-column 4096 tile leaves no room for a
// second buffer (passes.cu, p4096_r16x16x16_c4b1).  Here the tile being computed is held in
// REGISTERS (512 threads x 32 complex values = 128 KB of the 256 KB register file); shared memory
// holds only the next tile's TMA load (128 KB) and a half-tile exchange buffer (64 KB).  Each stage
// exchange runs in two halves: positions p < 2048 (the reader slots r' < 8) first, then the rest --
// with thread (f, j) owning butterflies j and j + 128 of column f, every writer writes exactly one
// butterfly per half in both exchanges (stage 0: p = 16 j + r; stage 1: p = (j div 16) 256 + j mod
// 16 + 16 r).  The last stage stores from registers straight to HBM: lanes walk 4 columns x 8
// outputs, so a later pass writes full 32-byte sectors of 8 strided rows per instruction, the first
// pass 64-byte runs of 4 contiguous columns.
//
// Measured on B200 (profiles/r02g): 2^22 as [4096, 1024] 1.78 ms and 2^23 as [4096, 2048] 1.93 ms
// per 2^28 elements (were 1.90 / 2.11 with the 2-column shared-memory 4096/2048 first pass); 2^24
// as two such passes ties the three 256-long passes (2.16-2.26 vs 2.21-2.23 ms).  Diagnosis (2^24,
// both passes, variants with parts removed): loads + stores alone 1.74 ms, arithmetic alone 1.34 ms
// -- the one tile in flight per SM streams at ~0.75 of the copy peak with 32-byte TMA rows, and the
// arithmetic of a 4096-long pass is itself ~0.67 ms per 2^28 elements, so the pair cannot reach the
// two-pass HBM bound (1.31 ms).  Variants tried and dropped: 16-byte cp.async per thread instead of
// the TMA boxes (2.98 ms), warp groups owning one or two columns each with named barriers (4.85 /
// 5.73 ms: their partial-sector strided stores double the DRAM traffic), stage twiddles copied to
// shared memory (2.25 ms), 2-column tiles at two CTAs per SM (6.5 ms).
#include <cuda.h>

#include "launch_util.h"
#include "passes.h"
#include "passtile.cuh"
#include "tma.cuh"

namespace fftc {

namespace {

constexpr int kL = 4096, kR = 16, kNB = kL / kR;  // 256 butterflies per column and stage
constexpr int kHalf = kL / 2;
constexpr int kC = 4;                              // columns per tile: 32-byte rows, full sectors
constexpr int kThreads = 512;
constexpr uint32_t kTileBytes = (uint32_t)kL * kC * 8u;

// exchange-buffer position of element p (mod 2048) of column f: 4 columns interleaved, the low 4
// bits of p XOR-swizzled with bits 4..7 -- conflict free for the radix-16 autosort writes (stride 1
// and 16 along r, lanes along j) and for the stage reads (lanes along j)
__device__ __forceinline__ int ex_idx(int p, int f) {
  return (((p & (kHalf - 16)) | ((p & 15) ^ ((p >> 4) & 15)))) * kC + f;
}

// Stockham write position of output r of butterfly j of a stage with Ns (L' = 16 Ns)
template <int Ns>
__device__ __forceinline__ int st_pos(int j, int r) {
  return (j / Ns) * (kR * Ns) + (j % Ns) + r * Ns;
}

// One exchange after the stage with Ns (1 or 16): v holds the stage outputs of butterflies jl
// (k = 0) and jl + 128 (k = 1); on return v holds the next stage's inputs x[j_k + 256 r].
template <int Ns>
__device__ __forceinline__ void exchange(float2* E, float2 (&v)[2][kR], int f, int jl) {
  float2 nv[2][kR];
  // half A: butterfly jl's outputs all have p < 2048
  sfor<kR>([&](auto r_) {
    constexpr int r = decltype(r_)::value;
    E[ex_idx(st_pos<Ns>(jl, r), f)] = v[0][r];
  });
  __syncthreads();
  sfor<2>([&](auto k_) {
    constexpr int k = decltype(k_)::value;
    const int b = ex_idx(jl + 128 * k, f);  // + 256 kC r' (bits 4..7 of p do not depend on r')
    sfor<kR / 2>([&](auto r_) {
      constexpr int r = decltype(r_)::value;
      nv[k][r] = E[b + r * (kNB * kC)];
    });
  });
  __syncthreads();
  // half B: butterfly jl + 128's outputs all have p >= 2048
  sfor<kR>([&](auto r_) {
    constexpr int r = decltype(r_)::value;
    E[ex_idx(st_pos<Ns>(jl + 128, r) - kHalf, f)] = v[1][r];
  });
  __syncthreads();
  sfor<2>([&](auto k_) {
    constexpr int k = decltype(k_)::value;
    const int b = ex_idx(jl + 128 * k, f);
    sfor<kR / 2>([&](auto r_) {
      constexpr int r = decltype(r_)::value;
      nv[k][r + kR / 2] = E[b + r * (kNB * kC)];
    });
  });
  sfor<2>([&](auto k_) {
    constexpr int k = decltype(k_)::value;
    sfor<kR>([&](auto r_) {
      constexpr int r = decltype(r_)::value;
      v[k][r] = nv[k][r];
    });
  });
}

// stage twiddles w_L'^{m r} (L' = 16 Ns) from the plan's stage table (entry (Ns - 1) + (r - 1) Ns + m):
// r = 1, 2, 4, 8 loaded, the others formed as products (as fused.cuh)
template <int Ns>
__device__ __forceinline__ void stage_tw(const float2* __restrict__ tw, int m, float2 (&w)[kR]) {
  const float2* t = tw + (Ns - 1) + m;
  sfor<kR - 1>([&](auto r_) {
    constexpr int r = decltype(r_)::value + 1;
    constexpr int hb = highbit(r);
    if constexpr (hb == r) w[r] = __ldg(t + (r - 1) * Ns);
    else w[r] = cmul(w[hb], w[r - hb]);
  });
}

// w[r] = u^r for r = 1..15 (a product tree, at most four roundings deep)
__device__ __forceinline__ void powers(float2 u, float2 (&w)[kR]) {
  w[1] = u;
  sfor<kR - 2>([&](auto r_) {
    constexpr int r = decltype(r_)::value + 2;
    constexpr int hb = highbit(r);
    w[r] = hb == r ? cmul(w[r / 2], w[r / 2]) : cmul(w[hb], w[r - hb]);
  });
}

// Persistent: one CTA of 512 threads per SM walks groups of adjacent 4-column tiles.  Thread
// (f = tid mod 4, jl = tid div 4) owns butterflies jl and jl + 128 of column f in every stage.
template <bool FIRST>
__global__ void __launch_bounds__(kThreads, 1)
    k_rpass(const __grid_constant__ CUtensorMap tin, float2* __restrict__ out, const float2* __restrict__ tw,
            const float2* __restrict__ twA, const float2* __restrict__ twB, PassGeom g, float csign_in,
            float csign_out) {
  extern __shared__ unsigned char smraw[];
  float2* A = reinterpret_cast<float2*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
  float2* E = A + kL * kC;
  __shared__ __align__(8) uint64_t full;
  const int f = (int)threadIdx.x % kC, jl = (int)threadIdx.x / kC;
  const long long T = g.tiles_total;
  const int tpb = g.tiles_per_batch;
  auto issue = [&](long long t) {  // the [4096 rows][4 columns] tile: 16 boxes of 256 rows
    const int b = (int)(t / tpb), c0 = (int)(t % tpb) * kC;
    mbar_arrive_expect_tx(&full, kTileBytes);
    sfor<kL / 256>([&](auto h_) {
      constexpr int h = decltype(h_)::value;
      tma_load_3d(A + h * 256 * kC, &tin, c0, h * 256, b, &full);
    });
  };
  if (threadIdx.x == 0) mbar_init(&full, 1);
  __syncthreads();
  const int grp = g.group;
  auto tile_of = [&](int i) -> long long {
    return ((long long)(i / grp) * gridDim.x + blockIdx.x) * grp + (i % grp);
  };
  if (threadIdx.x == 0 && tile_of(0) < T) issue(tile_of(0));
  const long long Ns = g.Ns;
  int it = 0;
  for (long long t = tile_of(0); t < T; t = tile_of(++it)) {
    const int b = (int)(t / tpb), c = (int)(t % tpb) * kC + f;
    float2 v[2][kR];
    // Input twiddle w_T^{m i} (T = Ns L, m = c mod Ns) of a later pass, folded into the three
    // stages: with i = j0 + 256 r0 (stage 0), j0 = (j1 div 16) + 16 r1 (stage 1) and j1 div 16 = r2
    // (stage 2), w^{m i} = (w^{256 m})^{r0} (w^{16 m})^{r1} (w^{m})^{r2}, so stage s multiplies its
    // input r by u_s^r with u_0 = w^{256 m}, u_1 = w^{16 m} w_256^{j1 mod 16}, u_2 = w^{m} w_4096^{j2}
    // -- the stage twiddles times a power of the column's root: powers of one value per stage and
    // butterfly, no separate input-twiddle multiply (the loads are issued before the tile wait).
    float2 om256, om16, om1, t1, t2[2];
    if constexpr (!FIRST) {
      const long long m = (long long)c % Ns;
      om256 = root_lookup_s(twA, twB, m * kNB, g.tws);
      om16 = root_lookup_s(twA, twB, m * 16, g.tws);
      om1 = root_lookup_s(twA, twB, m, g.tws);
      t1 = __ldg(tw + 15 + (jl & 15));     // w_256^{j1 mod 16}: stage-1 table, r = 1
      t2[0] = __ldg(tw + (kNB - 1) + jl);  // w_4096^{j2}: stage-2 table, r = 1
      t2[1] = __ldg(tw + (kNB - 1) + jl + 128);
    }
    mbar_wait(&full, it & 1);
    sfor<2>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      const float2* a = A + (jl + 128 * k) * kC + f;
      sfor<kR>([&](auto r_) {
        constexpr int r = decltype(r_)::value;
        float2 x = a[r * kNB * kC];
        if constexpr (FIRST) x.y *= csign_in;
        v[k][r] = x;
      });
    });
    fence_proxy_async_smem();
    __syncthreads();  // every thread has read the tile: the next one may stream into A
    if (threadIdx.x == 0 && tile_of(it + 1) < T) issue(tile_of(it + 1));
    {  // stage 0 (Ns = 1)
      float2 pw[kR];
      if constexpr (!FIRST) powers(om256, pw);
      sfor<2>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        if constexpr (!FIRST)
          sfor<kR - 1>([&](auto r_) {
            constexpr int r = decltype(r_)::value + 1;
            v[k][r] = cmul(v[k][r], pw[r]);
          });
        Codelet<kR>::run(v[k]);
      });
    }
    exchange<1>(E, v, f, jl);
    {  // stage 1 (Ns = 16): both butterflies share m = j mod 16
      float2 w[kR];
      if constexpr (FIRST) stage_tw<16>(tw, jl & 15, w);
      else powers(cmul(om16, t1), w);
      sfor<2>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        sfor<kR - 1>([&](auto r_) {
          constexpr int r = decltype(r_)::value + 1;
          v[k][r] = cmul(v[k][r], w[r]);
        });
        Codelet<kR>::run(v[k]);
      });
    }
    __syncthreads();  // the last half-B reads of exchange 1 precede exchange 2's writes
    exchange<16>(E, v, f, jl);
    // stage 2 (Ns = 256, m = j): outputs k = j + 256 r of column c, stored from registers
    float2* o;
    long long ostep;
    if constexpr (FIRST) {
      o = out + (long long)b * g.N + (long long)c * kL + jl;
      ostep = kNB;
    } else {
      o = out + (long long)b * g.N + (c / Ns) * Ns * kL + (c % Ns) + (long long)jl * Ns;
      ostep = kNB * Ns;
    }
    sfor<2>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      float2 w[kR];
      if constexpr (FIRST) stage_tw<kNB>(tw, jl + 128 * k, w);
      else powers(cmul(om1, t2[k]), w);
      sfor<kR - 1>([&](auto r_) {
        constexpr int r = decltype(r_)::value + 1;
        v[k][r] = cmul(v[k][r], w[r]);
      });
      Codelet<kR>::run(v[k]);
      float2* ok = o + (FIRST ? 128 * k : 128 * k * Ns);
      sfor<kR>([&](auto r_) {
        constexpr int r = decltype(r_)::value;
        __stcs(ok + r * ostep, make_float2(v[k][r].x, csign_out * v[k][r].y));
      });
    });
  }
}

}  // namespace

cudaError_t launch_rpass4096(bool first, const CUtensorMap& tin, const CUtensorMap&, float2* out, const float2* tw,
                             const float2* twA, const float2* twB, const PassGeom& g, int conj_in, int conj_out,
                             cudaStream_t st) {
  constexpr size_t smem = (size_t)(kL * kC + kHalf * kC) * sizeof(float2) + 128;
  static PerDevice<KernelSetup> ks_first_pd, ks_later_pd;
  const KernelSetup& ks = first ? ks_first_pd.get([&] { return kernel_setup(k_rpass<true>, kThreads, smem); })
                                : ks_later_pd.get([&] { return kernel_setup(k_rpass<false>, kThreads, smem); });
  if (ks.err != cudaSuccess) return ks.err;
  if (g.tiles_total == 0) return cudaSuccess;
  const long long groups = (g.tiles_total + g.group - 1) / g.group;
  const unsigned grid = (unsigned)(groups < ks.grid_max ? groups : ks.grid_max);
  auto kern = first ? k_rpass<true> : k_rpass<false>;
  kern<<<grid, kThreads, smem, st>>>(tin, out, tw, twA, twB, g, conj_in ? -1.f : 1.f, conj_out ? -1.f : 1.f);
  return cudaGetLastError();
}

}  // namespace fftc
