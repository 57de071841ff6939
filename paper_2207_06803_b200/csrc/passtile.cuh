// passtile.cuh -- one tile of a large-N Stockham pass (product path).
//
// A pass of length L is one level of the paper's Eq. 2 applied at the
// pass level (SURVEY App. A.2 with radix -> L):
//   column c < N/L, Ns = product of the earlier pass lengths:
//     v[r]  = a[c + r N/L]                                  (Pi folded into the column read)
//     v[r] *= w_{Ns L}^{(c mod Ns) r}          (Ns > 1)      (D^{Ns L}_{Ns})
//     v     = DFT_L v                                       (fused Stockham sub-stages, fused.cuh)
//     b[(c div Ns) Ns L + (c mod Ns) + r Ns] = v[r]
// A tile is C = 16 (or 8) adjacent columns held in shared memory as the TMA 128-byte
// (64-byte) swizzled [L rows][C columns] layout (LAY_TMA128 / LAY_TMA64).  pass_tile transforms it in place; both the
// HBM multi-pass kernels (passes.cu) and the L2-resident kernel (l2pass.cu) call it, so
// the two paths compute bit-identical results.
#pragma once
#include "colfft.cuh"

namespace fftc {

// DFT_L of the C columns of the tile, in place.  c = this thread's column (c0 + f);
// the input twiddle w_{Ns L}^{(c mod Ns) i} is applied when TW (every pass but the first), read
// as twA[e mod 2^tws] * twB[e >> tws] (tables built in double on the host).
// Shared-memory position of output k of column f for the first pass's TMA store: rows of 16
// consecutive outputs (128 B), row (k / 16) * C + f, 16-byte chunks XOR-swizzled by (f & 7) --
// the 128B-swizzled box [16 k][C columns][L / 16] of the (k % 16, c, k / 16, batch) view of a
// pass-0 output, where column c's L outputs are contiguous.
template <class P>
__device__ __forceinline__ int out0_idx(int f, int k) {
  return (((k >> 4) * P::FPB + f) << 4) + ((((k & 15) >> 1) ^ (f & 7)) << 1) + (k & 1);
}

// The input twiddles of one thread's sub-stage-0 butterfly (every pass kernel has one per
// thread: NB0 <= TPF): w^{m j} and the step powers w^{m NB0 2^b}.  They depend only on the
// column and the lane, so the kernels compute them before waiting for the tile's TMA load and
// the table latency hides under it.
struct PassTwPre {
  float2 sp[5];
  float2 base;
};
template <class P>
__device__ __forceinline__ PassTwPre pass_tw_pre(int c, int lt, int Ns, const float2* __restrict__ twA,
                                                 const float2* __restrict__ twB, int tws) {
  constexpr int L = P::N;
  constexpr int R0 = P::R(0);
  constexpr int NB0 = L / R0;
  constexpr int NB2 = ilog2(highbit(R0 - 1)) + 1;
  static_assert(NB2 <= 5 && NB0 <= P::TPF, "one sub-stage-0 butterfly per thread");
  PassTwPre t;
  const long long m = (long long)(c % Ns);
  t.sp[0] = root_lookup_s(twA, twB, m * NB0, tws);
  sfor<NB2 - 1>([&](auto b_) {
    constexpr int bb = decltype(b_)::value + 1;
    t.sp[bb] = cmul(t.sp[bb - 1], t.sp[bb - 1]);
  });
  t.base = lt < NB0 ? root_lookup_s(twA, twB, m * lt, tws) : make_float2(1.f, 0.f);
  return t;
}

// rmul / roff: the tile's row i is row rmul i + roff of the pass's column (a CTA of a cluster
// holding one residue class of the rows, cpass.cu); the input twiddle is w^{m (rmul i + roff)}.
template <class P, bool TW, bool OUT0 = false>
__device__ __forceinline__ void pass_tile(float2* sm, int f, int lt, int c, int Ns,
                                          const float2* __restrict__ tw, const float2* __restrict__ twA,
                                          const float2* __restrict__ twB, int tws, float csign_in,
                                          float csign_out, const PassTwPre* pre = nullptr, int rmul = 1,
                                          int roff = 0) {
  static_assert((P::FPB == 16 && P::LAY == LAY_TMA128) || (P::FPB == 8 && P::LAY == LAY_TMA64) ||
                    ((P::FPB == 2 || P::FPB == 4) && P::LAY == LAY_TMA16 && P::S >= 2),
                "pass tiles: 16 columns with the TMA 128B swizzle, 8 with the 64B swizzle, or 2/4 (linear)");
  constexpr int L = P::N;
  constexpr int R0 = P::R(0);
  constexpr int NB0 = L / R0;                      // sub-stage 0: element i = j + r NB0
  constexpr int NB2 = ilog2(highbit(R0 - 1)) + 1;  // step powers for r < R0
  // input twiddle w_T^{m i}, T = Ns L, m = c mod Ns: base per butterfly, step powers per thread
  const long long m = TW ? (long long)(c % Ns) : 0;
  float2 sp[NB2];
  if constexpr (TW) {
    if (pre) {
      sfor<NB2>([&](auto b_) {
        constexpr int bb = decltype(b_)::value;
        sp[bb] = pre->sp[bb];
      });
    } else {
      sp[0] = root_lookup_s(twA, twB, m * rmul * NB0, tws);
      sfor<NB2 - 1>([&](auto b_) {
        constexpr int bb = decltype(b_)::value + 1;
        sp[bb] = cmul(sp[bb - 1], sp[bb - 1]);
      });
    }
  }
  // input twiddles of one butterfly, formed as a tree: w[0] = base, w[r] = w[r - 2^b] sp[b]
  // (2^b = highest bit of r) -- one complex product per r, and the same product chain (lowest
  // bits first) as multiplying base by sp[b] for every set bit b of r
  float2 wt[R0];
  auto gload = [&](int i, int r, int pos) {
    float2 v = sm[pos];
    v.y *= csign_in;
    if constexpr (TW) {
      if (r == 0) {
        wt[0] = pre ? pre->base : root_lookup_s(twA, twB, m * ((long long)rmul * i + roff), tws);
      } else {
        int hb = 1, b = 0;
        while (2 * hb <= r) {
          hb *= 2;
          ++b;
        }
        wt[r] = cmul(wt[r - hb], sp[b]);
      }
      v = cmul(v, wt[r]);
    }
    return v;
  };
  // the last sub-stage writes in place (all reads precede it); OUT0: in the pass-0 store layout
  auto gstore = [&](int i, float2 v, int, int pos) {
    if constexpr (OUT0) sm[out0_idx<P>(f, i)] = make_float2(v.x, csign_out * v.y);
    else sm[pos] = make_float2(v.x, csign_out * v.y);
  };
  // sub-stages of DFT_L in place on the tile (every stage reads all, syncs, writes)
  sfor<P::S>([&](auto s_) {
    constexpr int s = decltype(s_)::value;
    stage<P, s, s == 0, s == P::S - 1, true>(sm, f, lt, true, tw, gload, gstore);
  });
}

// First pass (Ns = 1): column c's L outputs are contiguous at c L + r; go = base + c0 L.
// Lanes walk r (coalesced 8-byte stores through st(ptr, value)).  Caller syncs before.
template <class P, class ST>
__device__ __forceinline__ void pass0_store(const float2* sm, float2* __restrict__ go, ST&& st) {
  constexpr int L = P::N, C = P::FPB;
  if constexpr (P::LAY == LAY_TMA128 && L <= 128) {
    // columns 2q and 2q+1 of row r share one 16-byte chunk (q ^ (r & 7)) of the swizzled row:
    // one conflict-free 128-bit shared load per pair, two coalesced stores (lanes walk r).
    // Measured (same box A/B): 2^13 1.56 -> 1.52 ms; slower for L = 256 (2^16 1.50 -> 1.54 ms),
    // which keeps the one-column-per-instruction walk below.  Its shared reads are 2-way
    // conflicted (lanes repeat r & 7); a conflict-free walk (a warp = 16 rows x 2 columns,
    // two full 128-byte lines per store) measured slower still: 2^16 1.49 -> 1.52 ms.
    constexpr int PER = L * (C / 2) / P::THREADS;
    static_assert((L * (C / 2)) % P::THREADS == 0, "tile must split evenly");
    sfor<PER>([&](auto n_) {
      constexpr int n = decltype(n_)::value;
      const int e = threadIdx.x + n * P::THREADS;
      const int r = e % L, q = e / L;
      const float4 v = *reinterpret_cast<const float4*>(sm + r * 16 + ((q ^ (r & 7)) << 1));
      st(go + (2 * q) * L + r, make_float2(v.x, v.y));
      st(go + (2 * q + 1) * L + r, make_float2(v.z, v.w));
    });
  } else {
    constexpr int PER = L * C / P::THREADS;
    static_assert((L * C) % P::THREADS == 0, "tile must split evenly");
    sfor<PER>([&](auto n_) {
      constexpr int n = decltype(n_)::value;
      const int e = threadIdx.x + n * P::THREADS;
      const int r = e % L, cc = e / L;
      st(go + cc * L + r, sm[P::lidx(cc, r)]);
    });
  }
}

}  // namespace fftc
