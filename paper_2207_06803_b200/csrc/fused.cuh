// fused.cuh -- single-pass fused Stockham kernels for sm_100a (product path).
//
// One kernel computes whole DFT_N's (N <= 4096) for a tile of FPB transforms:
// stage-in, S Stockham stages, stage-out; nothing but the input and output
// touches HBM.  Stage s (radix R, Ns = R_0...R_{s-1}, L = Ns R) is one level of
// the paper's Eq. 2 with (N -> L, K -> R, M -> Ns):
//   for each butterfly j in [0, N/R):
//     v[r]  = a[j + r N/R]                           (Pi folded into the read stride)
//     v[r] *= w_L^{(j mod Ns) r}        (s > 0)      (D^L_Ns, fp32 table from double)
//     v     = DFT_R v                                (register codelet, codelets.cuh)
//     b[(j div Ns) L + (j mod Ns) + r Ns] = v[r]     (Stockham autosort: natural order out)
// Stages exchange through shared memory in place: every thread first reads all
// of its butterflies' inputs into registers, the group barrier-syncs, then
// writes.  Index maps verified against numpy in DESIGN.md §5 / tests.
//
// Thread mappings (Map):
//   LT_FAST: tid = f*TPF + lt -- lanes walk one transform (large N).  Stage 0 can
//            read HBM directly (coalesced along j) and the last stage can write
//            HBM directly (coalesced along j).  Shared layout f*N + swz(i), swz an
//            XOR swizzle of the low 4 bits of i by bits 4..7 (bank-conflict free for
//            the power-of-two write strides of the autosort).
//   F_FAST : tid = lt*FPB + f -- lanes walk transforms (small N).  I/O is staged
//            through shared memory with contiguous 128-bit copies; shared layout
//            f*(N|1) + i (odd stride -> conflict free across transforms).
#pragma once
#include <stdlib.h>

#include <type_traits>

#include "codelets.cuh"
#include "launch_util.h"
#include "tma.cuh"

namespace fftc {

enum Map : int { LT_FAST = 0, F_FAST = 1 };

#ifndef FFTC_TW_LOAD_ALL
#define FFTC_TW_LOAD_ALL 0  // measured on B200: loading every twiddle is slower (L1-bound): 3125 199 -> 216 us
#endif
constexpr bool kTwLoadAll = FFTC_TW_LOAD_ALL != 0;

constexpr int highbit(int r) {
  int h = 1;
  while (h * 2 <= r) h *= 2;
  return h;
}

template <int... Rs>
struct Radices {
  static constexpr int S = sizeof...(Rs);
  static constexpr int R[S] = {Rs...};
  static constexpr int prod() {
    int p = 1;
    for (int s = 0; s < S; ++s) p *= R[s];
    return p;
  }
  static constexpr int ns(int s) {
    int p = 1;
    for (int t = 0; t < s; ++t) p *= R[t];
    return p;
  }
};

// Shared-memory layouts of a tile of FPB transforms (element i of transform f):
//   LAY_SWZ  : f*SS + swz(i), swz XORs bits 0..3 of i with bits 4..7 (LT_FAST; lanes
//              of a 16-lane phase walk one transform; power-of-two autosort strides).
//   LAY_FXOR : f*N + (i ^ gf(f)) (F_FAST, N % 16 == 0 or N == 8; lanes walk f).
//   LAY_ODD  : f*SS + i, SS odd (F_FAST, other N).
//   LAY_INTER: swzc(i)*FPB + f (interleaved columns, F_FAST with FPB < 16: a phase
//              holds FPB columns x 16/FPB consecutive butterflies).
//   LAY_TMA64: i*8 + (((f >> 1) ^ ((i >> 1) & 3)) << 1 | (f & 1)) -- the TMA 64-byte swizzle of a
//              [row i][8 columns] complex64 tile (512-byte aligned), FPB = 8.
//   LAY_TMA128: i*16 + (((f >> 1) ^ (i & 7)) << 1 | (f & 1)) -- the TMA 128-byte swizzle of a
//              [row i][16 columns] complex64 tile (1024-byte aligned), FPB = 16.
//   LAY_PAD16: f*SS + i + (i >> PSH), SS = N + (N >> PSH), PSH = log2 of 16, or of 32 when the leaf
//              radix R_0 >= 32 (LT_FAST, N % 16 == 0): one pad element per 16 (32) elements.
//              For the power-of-two Stockham accesses (reads j + r NB, writes o + r Ns with
//              compile-time r) the padded position is (base of j) + (compile-time offset of r), so
//              the addresses need no per-element XOR; lanes walking j stay bank-conflict free.
//   LAY_TMA16: 2- or 4-column tiles of long passes (16/32-byte TMA rows, no swizzle).  The
//              TMA-facing layout (first reads, last writes: `lidx`) is linear, i*FPB + f; the
//              in-between stage exchanges XOR the low log2(16/FPB) bits of i with the bits from 4
//              up (`sidx`), which keeps the radix-16 autosort writes conflict free.
enum Layout : int { LAY_AUTO = -1, LAY_SWZ = 0, LAY_FXOR = 1, LAY_ODD = 2, LAY_INTER = 3, LAY_TMA128 = 4, LAY_TMA64 = 5,
                    LAY_TMA16 = 6, LAY_PAD16 = 7 };

constexpr int ilog2(int n) {
  int l = 0;
  while ((1 << (l + 1)) <= n) ++l;
  return l;
}

// Compile-time schedule of one fused transform.
//   N: length, Rad: Radices<...>, TPF: threads per transform, FPB: transforms per CTA,
//   MAP: thread mapping, PAD: extra elements per transform row (LAY_SWZ / LAY_ODD).
//   TAG: distinguishes otherwise identical schedules compiled in another translation unit with
//   different codelet arithmetic (kernels_packed.cu), so their kernel symbols stay distinct.
// Schedule options (OPT bit mask; each variant is its own kernel instantiation):
//   OPT_TW_LOAD  : every stage twiddle w_L^{m r} is loaded from the table (else r = 2^b loaded,
//                  the other r formed as products, the default for power-of-two radices)
//   OPT_VEC_IO   : direct HBM I/O stages assign each thread PAIRS of adjacent butterflies
//                  (j = 2p, 2p + 1) and move both with one 128-bit load / store per r
//   OPT_TW_SHARE : when TPF is a multiple of Ns, a thread's butterflies of a stage share
//                  m = j mod Ns, so their twiddles are formed once per thread, not per butterfly
//   OPT_LD_NA    : direct HBM loads with ld.global.nc.L1::no_allocate (the streamed input does not
//                  displace the L1-resident twiddle tables)
enum SchedOpt : int { OPT_TW_LOAD = 1, OPT_VEC_IO = 2, OPT_TW_SHARE = 4, OPT_LD_NA = 8 };

__device__ __forceinline__ float2 ld_na(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

template <int N_, class Rad, int TPF_, int FPB_, int MAP_, int PAD_ = 0, int LAY_ = LAY_AUTO, int TAG_ = 0,
          int OPT_ = 0>
struct Sched {
  static constexpr int N = N_, TPF = TPF_, FPB = FPB_, MAP = MAP_, OPT = OPT_;
  static constexpr int S = Rad::S;
  static constexpr int THREADS = TPF * FPB;
  static_assert(Rad::prod() == N, "radices must multiply to N");
  static_assert(THREADS <= 1024, "too many threads");
  static constexpr int R(int s) { return Rad::R[s]; }
  static constexpr int ns(int s) { return Rad::ns(s); }
  static constexpr int LAY = (LAY_ != LAY_AUTO) ? LAY_
                             : (MAP == LT_FAST) ? LAY_SWZ
                             : (PAD_ == 0 && (N % 16 == 0 || N == 8)) ? LAY_FXOR : LAY_ODD;
  static constexpr bool FXOR = (LAY == LAY_FXOR);
  static constexpr bool SWZ = (LAY == LAY_SWZ) && ((N + PAD_) % 16 == 0);
  static_assert(LAY != LAY_PAD16 || (N % 16 == 0 && PAD_ == 0), "LAY_PAD16: N a multiple of 16");
  // LAY_PAD16 period: the leaf stage writes j R_0 + r, conflict free when the period is R_0
  static constexpr int PSH = (Rad::R[0] >= 32 && N % 32 == 0) ? 5 : 4;
  static constexpr int SS = (LAY == LAY_FXOR) ? N : (LAY == LAY_ODD) ? ((N + PAD_) | 1)
                            : (LAY == LAY_PAD16) ? (N + (N >> PSH)) : (N + PAD_);
  static constexpr size_t SMEM = size_t(LAY == LAY_INTER ? N : SS) * FPB * sizeof(float2);
  // LAY_INTER: XOR the bank bits of i (mod 16/FPB) with the bits above the leaf radix
  static constexpr int IMASK = (LAY == LAY_INTER && FPB < 16) ? (16 / FPB - 1) : 0;
  static constexpr int ISHIFT = ilog2(Rad::R[0]);
  // a transform's threads share one warp -> warp-level barrier suffices
  static constexpr bool WARP_SYNC = (MAP == LT_FAST) && (TPF <= 32) && (32 % TPF == 0);
  FFTC_HD static int swz(int i) { return SWZ ? (i ^ ((i >> 4) & 15)) : i; }
  FFTC_HD static int gf(int f) { return (N % 16 == 0) ? (f & 15) : ((f >> 1) & 7); }
  FFTC_HD static int sidx(int f, int i) {
    if constexpr (LAY == LAY_FXOR) return f * SS + (i ^ gf(f));
    else if constexpr (LAY == LAY_TMA128) return i * 16 + ((((f >> 1) ^ (i & 7)) << 1) | (f & 1));
    else if constexpr (LAY == LAY_TMA64) return i * 8 + ((((f >> 1) ^ ((i >> 1) & 3)) << 1) | (f & 1));
    else if constexpr (LAY == LAY_TMA16) return ((i ^ ((i >> 4) & (16 / FPB - 1))) * FPB) | f;
    else if constexpr (LAY == LAY_INTER) return (i ^ ((i >> ISHIFT) & IMASK)) * FPB + f;
    else if constexpr (LAY == LAY_PAD16) return f * SS + i + (i >> PSH);
    else return f * SS + swz(i);
  }
  // sidx(f, i0 + D) from pos0 = sidx(f, i0) for a compile-time D, with no per-element index math
  // where the layout makes it linear: LAY_PAD16 when D is a multiple of the pad period, or when i0
  // is (I0_ALIGNED) and D is any offset; LAY_SWZ when D is a multiple of 256 (bits 4..7 unchanged)
  template <int D, bool I0_ALIGNED>
  FFTC_HD static int sidx_plus(int f, int i0, int pos0) {
    if constexpr (LAY == LAY_PAD16 && (D % (1 << PSH) == 0 || I0_ALIGNED)) return pos0 + D + (D >> PSH);
    else if constexpr (LAY == LAY_SWZ && SWZ && D % 256 == 0) return pos0 + D;
    else if constexpr ((LAY == LAY_SWZ && !SWZ) || LAY == LAY_ODD) return pos0 + D;  // f SS + i
    else if constexpr (LAY == LAY_TMA128 && D % 8 == 0) return pos0 + D * 16;  // (i & 7) unchanged
    else if constexpr (LAY == LAY_TMA64 && D % 8 == 0) return pos0 + D * 8;    // (i >> 1) & 3 unchanged
    else if constexpr (LAY == LAY_TMA16 && D % 128 == 0) return pos0 + D * FPB;  // i >> 4 & (16/FPB-1) unchanged
    else return sidx(f, i0 + D);
  }
  // lidx(f, i0 + D) from pos0 = lidx(f, i0), as sidx_plus (LAY_TMA16's TMA-facing rows are linear)
  template <int D, bool I0_ALIGNED>
  FFTC_HD static int lidx_plus(int f, int i0, int pos0) {
    if constexpr (LAY == LAY_TMA16) return pos0 + D * FPB;
    else return sidx_plus<D, I0_ALIGNED>(f, i0, pos0);
  }
  // position of element i of column f in the layout the TMA reads and writes (= sidx except
  // for LAY_TMA16, whose exchanges are swizzled but whose TMA rows are linear)
  FFTC_HD static int lidx(int f, int i) {
    if constexpr (LAY == LAY_TMA16) return i * FPB + f;
    else return sidx(f, i);
  }
  __device__ __forceinline__ static void sync() {
    if constexpr (WARP_SYNC) __syncwarp();
    else __syncthreads();
  }
  __device__ __forceinline__ static void thread_coords(int tid, int& f, int& lt) {
    if constexpr (MAP == LT_FAST) {
      f = tid / TPF;
      lt = tid % TPF;
    } else {
      f = tid % FPB;
      lt = tid / FPB;
    }
  }
};

// One Stockham stage.  SRC_G: stage reads through gload(i, r) (HBM, or a staging
// buffer); DST_G: stage writes through gstore(i, v, r) (HBM, or shared memory in
// the transposed-output column kernel: then MID_SYNC forces the in-place barrier
// between the reads and the writes); r = the element's index within its butterfly.
// gload2(i) / gstore2(i, a, b): elements i and i + 1 at once (OPT_VEC_IO stages only).
// Twiddle table layout (per plan, built on the host in double): stage s occupies
// entries [Ns-1, Ns-1 + (R-1) Ns), entry (Ns-1) + (r-1) Ns + m = w_L^{m r}.
template <class P, int s, bool SRC_G, bool DST_G, bool MID_SYNC, class GL, class GS, class GL2, class GS2>
__device__ __forceinline__ void stage_io(float2* sm, int f, int lt, bool fvalid, const float2* __restrict__ tw,
                                         GL&& gload, GS&& gstore, GL2&& gload2, GS2&& gstore2) {
  constexpr int R = P::R(s);
  constexpr int NB = P::N / R;
  constexpr int Ns = P::ns(s);
  constexpr int L = Ns * R;
  constexpr int KB = (NB + P::TPF - 1) / P::TPF;
  constexpr bool EXACT = (NB % P::TPF) == 0;
  // paired mapping for a direct-I/O stage: thread lt, pair k/2 -> butterflies j = 2p, 2p + 1
  constexpr bool VEC = (P::OPT & OPT_VEC_IO) && (SRC_G || DST_G) && (KB % 2 == 0) && (NB % (2 * P::TPF) == 0) &&
                      (!DST_G || Ns % 2 == 0);
  // butterflies of one thread share m = j mod Ns (strided mapping, TPF a multiple of Ns)
  constexpr bool SHARE = (P::OPT & OPT_TW_SHARE) && !VEC && s > 0 && KB > 1 && (P::TPF % Ns == 0);
  constexpr bool LOAD_ALL = (P::OPT & OPT_TW_LOAD) || (kTwLoadAll && (R & (R - 1)) != 0);
  auto bfly = [&](int k) { return VEC ? 2 * (lt + (k >> 1) * P::TPF) + (k & 1) : lt + k * P::TPF; };
  float2 v[KB][R];
  if constexpr (VEC && SRC_G) {
    sfor<KB / 2>([&](auto k_) {
      constexpr int k = 2 * decltype(k_)::value;
      const int j = bfly(k);
      if (fvalid)
        sfor<R>([&](auto r_) {
          constexpr int r = decltype(r_)::value;
          const float4 q = gload2(j + r * NB);
          v[k][r] = make_float2(q.x, q.y);
          v[k + 1][r] = make_float2(q.z, q.w);
        });
    });
  } else {
    sfor<KB>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      const int j = bfly(k);
      if (fvalid && (EXACT || j < NB)) {
        constexpr bool GPOS = SRC_G && std::is_invocable_v<GL, int, int, int>;  // gload(i, r, lidx position)
        const int p0 = SRC_G ? (GPOS ? P::lidx(f, j) : 0) : P::sidx(f, j);
        sfor<R>([&](auto r_) {
          constexpr int r = decltype(r_)::value;
          const int i = j + r * NB;
          if constexpr (GPOS) v[k][r] = gload(i, r, P::template lidx_plus<r * NB, false>(f, j, p0));
          else if constexpr (SRC_G) v[k][r] = gload(i, r);
          else v[k][r] = sm[P::template sidx_plus<r * NB, false>(f, j, p0)];
        });
      }
    });
  }
  if constexpr ((!SRC_G && !DST_G) || MID_SYNC) P::sync();
  // w_L^{m r}: power-of-two radices load r = 1, 2, 4, 8, ... from the table and form every other
  // r as the product w^{2^b} w^{r - 2^b} (at most log2(R)-1 roundings deep); LOAD_ALL loads all
  auto twiddles = [&](int m, float2* w) {
    const float2* t = tw + (Ns - 1) + m;
    sfor<R - 1>([&](auto r_) {
      constexpr int r = decltype(r_)::value + 1;
      constexpr int hb = highbit(r);
      if constexpr (LOAD_ALL || hb == r) w[r] = __ldg(t + (r - 1) * Ns);
      else w[r] = cmul(w[hb], w[r - hb]);
    });
  };
  if constexpr (SHARE) {
    if (fvalid) {
      float2 w[R];
      twiddles(lt % Ns, w);
      sfor<KB>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        if (EXACT || bfly(k) < NB)
          sfor<R - 1>([&](auto r_) {
            constexpr int r = decltype(r_)::value + 1;
            v[k][r] = cmul(v[k][r], w[r]);
          });
      });
    }
  }
  sfor<KB>([&](auto k_) {
    constexpr int k = decltype(k_)::value;
    const int j = bfly(k);
    if (fvalid && (EXACT || j < NB)) {
      const int m = (Ns == 1) ? 0 : (j % Ns);
      if constexpr (s > 0 && !SHARE) {
        float2 w[R];
        twiddles(m, w);
        sfor<R - 1>([&](auto r_) {
          constexpr int r = decltype(r_)::value + 1;
          v[k][r] = cmul(v[k][r], w[r]);
        });
      }
      Codelet<R>::run(v[k]);
      if constexpr (!(VEC && DST_G)) {
        const int o = (Ns == 1) ? j * R : ((j / Ns) * L + m);
        // o = j R is a multiple of the LAY_PAD16 period when R is
        constexpr bool OALIGNED = (Ns == 1) && (R % (1 << P::PSH) == 0);
        constexpr bool SPOS = DST_G && std::is_invocable_v<GS, int, float2, int, int>;  // gstore(i, v, r, lidx pos)
        const int q0 = DST_G ? (SPOS ? P::lidx(f, o) : 0) : P::sidx(f, o);
        sfor<R>([&](auto r_) {
          constexpr int r = decltype(r_)::value;
          if constexpr (SPOS) gstore(o + r * Ns, v[k][r], r, P::template lidx_plus<r * Ns, OALIGNED>(f, o, q0));
          else if constexpr (DST_G) gstore(o + r * Ns, v[k][r], r);
          else sm[P::template sidx_plus<r * Ns, OALIGNED>(f, o, q0)] = v[k][r];
        });
      }
    }
  });
  if constexpr (VEC && DST_G) {
    // the pair's outputs o + r Ns and o + 1 + r Ns are adjacent when Ns > 1 (m and m + 1 < Ns)
    static_assert(Ns % 2 == 0, "paired stores need an even Ns");
    sfor<KB / 2>([&](auto k_) {
      constexpr int k = 2 * decltype(k_)::value;
      const int j = bfly(k);
      if (fvalid) {
        const int o = (j / Ns) * L + (j % Ns);
        sfor<R>([&](auto r_) {
          constexpr int r = decltype(r_)::value;
          gstore2(o + r * Ns, v[k][r], v[k + 1][r]);
        });
      }
    });
  }
  if constexpr (!DST_G) P::sync();
}

template <class P, int s, bool SRC_G, bool DST_G, bool MID_SYNC = false, class GL, class GS>
__device__ __forceinline__ void stage(float2* sm, int f, int lt, bool fvalid, const float2* __restrict__ tw,
                                      GL&& gload, GS&& gstore) {
  stage_io<P, s, SRC_G, DST_G, MID_SYNC>(
      sm, f, lt, fvalid, tw, gload, gstore, [](int) { return make_float4(0.f, 0.f, 0.f, 0.f); },
      [](int, float2, float2) {});
}

// All S stages.  SRC0_G: stage 0 reads HBM; DSTL_G: the last stage writes through
// gstore; LAST_MID: the last stage's gstore writes the shared exchange buffer.
template <class P, bool SRC0_G, bool DSTL_G, bool LAST_MID = false, class GL, class GS>
__device__ __forceinline__ void run_stages(float2* sm, int f, int lt, bool fvalid,
                                           const float2* __restrict__ tw, GL&& gload, GS&& gstore) {
  sfor<P::S>([&](auto s_) {
    constexpr int s = decltype(s_)::value;
    stage<P, s, SRC0_G && s == 0, DSTL_G && s == P::S - 1, LAST_MID && s == P::S - 1>(sm, f, lt, fvalid, tw, gload,
                                                                                        gstore);
  });
}

template <class P, class GL, class GS, class GL2, class GS2>
__device__ __forceinline__ void run_stages_io(float2* sm, int f, int lt, bool fvalid, const float2* __restrict__ tw,
                                              GL&& gload, GS&& gstore, GL2&& gload2, GS2&& gstore2) {
  sfor<P::S>([&](auto s_) {
    constexpr int s = decltype(s_)::value;
    stage_io<P, s, s == 0, s == P::S - 1, false>(sm, f, lt, fvalid, tw, gload, gstore, gload2, gstore2);
  });
}

// Contiguous HBM tile <-> shared (layout P::sidx), 128-bit when the tile base is
// 16-byte aligned (FPB*N even), element-wise for ragged tails.  csign = -1 applies
// the conjugation of the inverse transform (IDFT x = conj DFT conj x).
template <class P>
__device__ __forceinline__ void tile_in(float2* sm, const float2* __restrict__ g, int nf, float csign) {
  constexpr int N = P::N;
  constexpr int TOTAL = P::FPB * N;
  if constexpr (P::FXOR) {
    // 128-bit loads, 128-bit stores into the XOR layout (pairs stay aligned, maybe swapped)
    if (nf == P::FPB) {
      constexpr int PAIRS = TOTAL / 2;
      constexpr int PER = (PAIRS + P::THREADS - 1) / P::THREADS;
      const float4* g4 = reinterpret_cast<const float4*>(g);
      float4 q[PER];
      sfor<PER>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int p = threadIdx.x + k * P::THREADS;
        if (PAIRS % P::THREADS == 0 || p < PAIRS) q[k] = __ldcs(g4 + p);
      });
      sfor<PER>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int p = threadIdx.x + k * P::THREADS;
        if (PAIRS % P::THREADS == 0 || p < PAIRS) {
          const int e = 2 * p, f = e / N, i = e % N, gx = P::gf(f);
          float4 v = make_float4(q[k].x, csign * q[k].y, q[k].z, csign * q[k].w);
          if (gx & 1) v = make_float4(v.z, v.w, v.x, v.y);
          *reinterpret_cast<float4*>(sm + f * N + ((i ^ gx) & ~1)) = v;
        }
      });
      return;
    }
  } else if constexpr (TOTAL % 2 == 0 && P::MAP == LT_FAST) {
    if (nf == P::FPB) {
      constexpr int PAIRS = TOTAL / 2;
      constexpr int PER = (PAIRS + P::THREADS - 1) / P::THREADS;
      const float4* g4 = reinterpret_cast<const float4*>(g);
      float4 q[PER];
      sfor<PER>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int p = threadIdx.x + k * P::THREADS;
        if (PAIRS % P::THREADS == 0 || p < PAIRS) q[k] = __ldcs(g4 + p);
      });
      sfor<PER>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int p = threadIdx.x + k * P::THREADS;
        if (PAIRS % P::THREADS == 0 || p < PAIRS) {
          const int e = 2 * p;
          sm[P::sidx(e / N, e % N)] = make_float2(q[k].x, csign * q[k].y);
          sm[P::sidx((e + 1) / N, (e + 1) % N)] = make_float2(q[k].z, csign * q[k].w);
        }
      });
      return;
    }
  } else {
    // odd shared stride: element-wise (consecutive lanes -> consecutive banks)
    if (nf == P::FPB) {
      constexpr int PER = (TOTAL + P::THREADS - 1) / P::THREADS;
      float2 q[PER];
      sfor<PER>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int e = threadIdx.x + k * P::THREADS;
        if (TOTAL % P::THREADS == 0 || e < TOTAL) q[k] = __ldcs(g + e);
      });
      sfor<PER>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int e = threadIdx.x + k * P::THREADS;
        if (TOTAL % P::THREADS == 0 || e < TOTAL) sm[P::sidx(e / N, e % N)] = make_float2(q[k].x, csign * q[k].y);
      });
      return;
    }
  }
  const int total = nf * N;
  for (int e = threadIdx.x; e < total; e += P::THREADS) {
    float2 a = __ldcs(g + e);
    sm[P::sidx(e / N, e % N)] = make_float2(a.x, csign * a.y);
  }
}

template <class P>
__device__ __forceinline__ void tile_out(const float2* sm, float2* __restrict__ g, int nf, float csign) {
  constexpr int N = P::N;
  constexpr int TOTAL = P::FPB * N;
  if constexpr (P::FXOR) {
    if (nf == P::FPB) {
      constexpr int PAIRS = TOTAL / 2;
      constexpr int PER = (PAIRS + P::THREADS - 1) / P::THREADS;
      float4* g4 = reinterpret_cast<float4*>(g);
      sfor<PER>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int p = threadIdx.x + k * P::THREADS;
        if (PAIRS % P::THREADS == 0 || p < PAIRS) {
          const int e = 2 * p, f = e / N, i = e % N, gx = P::gf(f);
          float4 v = *reinterpret_cast<const float4*>(sm + f * N + ((i ^ gx) & ~1));
          if (gx & 1) v = make_float4(v.z, v.w, v.x, v.y);
          __stcs(g4 + p, make_float4(v.x, csign * v.y, v.z, csign * v.w));
        }
      });
      return;
    }
  } else if constexpr (TOTAL % 2 == 0 && P::MAP == LT_FAST) {
    if (nf == P::FPB) {
      constexpr int PAIRS = TOTAL / 2;
      constexpr int PER = (PAIRS + P::THREADS - 1) / P::THREADS;
      float4* g4 = reinterpret_cast<float4*>(g);
      sfor<PER>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int p = threadIdx.x + k * P::THREADS;
        if (PAIRS % P::THREADS == 0 || p < PAIRS) {
          const int e = 2 * p;
          float2 a = sm[P::sidx(e / N, e % N)];
          float2 b = sm[P::sidx((e + 1) / N, (e + 1) % N)];
          __stcs(g4 + p, make_float4(a.x, csign * a.y, b.x, csign * b.y));
        }
      });
      return;
    }
  } else {
    if (nf == P::FPB) {
      constexpr int PER = (TOTAL + P::THREADS - 1) / P::THREADS;
      sfor<PER>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int e = threadIdx.x + k * P::THREADS;
        if (TOTAL % P::THREADS == 0 || e < TOTAL) {
          float2 a = sm[P::sidx(e / N, e % N)];
          __stcs(g + e, make_float2(a.x, csign * a.y));
        }
      });
      return;
    }
  }
  const int total = nf * N;
  for (int e = threadIdx.x; e < total; e += P::THREADS) {
    float2 a = sm[P::sidx(e / N, e % N)];
    __stcs(g + e, make_float2(a.x, csign * a.y));
  }
}

// ---------------------------------------------------------------- batched kernel
// DIRECT: stage 0 loads HBM and the last stage stores HBM (LT_FAST only);
// otherwise tile_in / tile_out stage the contiguous FPB*N tile through shared.
template <class P, bool DIRECT, int MINB>
__global__ void __launch_bounds__(P::THREADS, MINB)
    k_fused_batch(const float2* __restrict__ in, float2* __restrict__ out,
                  const float2* __restrict__ tw, long long batch, float csign) {
  extern __shared__ float2 sm[];
  int f, lt;
  P::thread_coords(threadIdx.x, f, lt);
  const long long f0 = (long long)blockIdx.x * P::FPB;
  const long long rem = batch - f0;
  const int nf = rem < P::FPB ? (int)rem : P::FPB;
  const bool fvalid = f < nf;
  const float2* gin = in + f0 * P::N;
  float2* gout = out + f0 * P::N;
  if constexpr (DIRECT) {
    static_assert(P::MAP == LT_FAST, "direct I/O needs the LT_FAST mapping");
    const float2* gi = gin + (long long)f * P::N;
    float2* go = gout + (long long)f * P::N;
    run_stages_io<P>(
        sm, f, lt, fvalid, tw,
        [&](int i, int) {
          float2 a = (P::OPT & OPT_LD_NA) ? ld_na(gi + i) : __ldcs(gi + i);
          return make_float2(a.x, csign * a.y);
        },
        [&](int i, float2 v, int) { __stcs(go + i, make_float2(v.x, csign * v.y)); },
        [&](int i) {  // OPT_VEC_IO: i even, the row 16-byte aligned (N even, checked base)
          float4 q = __ldcs(reinterpret_cast<const float4*>(gi + i));
          return make_float4(q.x, csign * q.y, q.z, csign * q.w);
        },
        [&](int i, float2 a, float2 b) {
          __stcs(reinterpret_cast<float4*>(go + i), make_float4(a.x, csign * a.y, b.x, csign * b.y));
        });
  } else {
    tile_in<P>(sm, gin, nf, csign);
    __syncthreads();
    run_stages<P, false, false>(
        sm, f, lt, fvalid, tw, [&](int, int) { return make_float2(0.f, 0.f); }, [&](int, float2, int) {});
    __syncthreads();
    tile_out<P>(sm, gout, nf, 1.0f * csign);
  }
}

// Host launcher for one compiled schedule.
template <class P, bool DIRECT, int MINB>
static cudaError_t launch_fused_batch(const float2* in, float2* out, const float2* tw, long long batch,
                                      int conj, cudaStream_t st) {
  auto kern = k_fused_batch<P, DIRECT, MINB>;
  static PerDevice<cudaError_t> attr_pd;
  const cudaError_t attr = attr_pd.get([&] {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::SMEM);
    // FFTC_CARVEOUT=<percent> (tuning): the shared-memory share of the unified L1/shared array,
    // i.e. how much L1 stays for in-flight loads; default: the driver's choice
    if (const char* c = getenv("FFTC_CARVEOUT"))
      if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(c));
    return e;
  });
  if (attr != cudaSuccess) return attr;
  const long long grid = (batch + P::FPB - 1) / P::FPB;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)grid, P::THREADS, P::SMEM, st>>>(in, out, tw, batch, conj ? -1.0f : 1.0f);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- warp-shuffle exchange (A/B variant)
// N = R * R with TPF = R lanes per transform (R <= 32, a power of two), two Stockham stages.
// Stage 0's butterfly j = lt writes positions R lt + r; stage 1's butterfly j = lt reads
// positions lt + R r = element lt of lane r: the exchange is an R x R transpose across the
// transform's R lanes, done here in registers by log2(R) shfl.xor rounds (round mask m: each lane
// keeps the elements whose index bit m equals its own lane bit and swaps the other half with lane
// lt ^ m) instead of through shared memory.  Same twiddles, codelets and order of arithmetic as
// the shared-memory kernel, so the results are bit-identical; no shared memory, no barrier.
template <int R>
__device__ __forceinline__ void lane_transpose(float2 (&v)[R], int lt) {
  sfor<ilog2(R)>([&](auto b_) {
    constexpr int m = 1 << decltype(b_)::value;
    const bool hi = (lt & m) != 0;
    sfor<R>([&](auto r_) {
      constexpr int r = decltype(r_)::value;
      if constexpr ((r & m) == 0) {
        const float2 send = hi ? v[r] : v[r | m];
        float2 recv;
        recv.x = __shfl_xor_sync(0xffffffffu, send.x, m);
        recv.y = __shfl_xor_sync(0xffffffffu, send.y, m);
        if (hi) v[r] = recv;
        else v[r | m] = recv;
      }
    });
  });
}

template <class P, int MINB>
__global__ void __launch_bounds__(P::THREADS, MINB)
    k_fused_shfl(const float2* __restrict__ in, float2* __restrict__ out, const float2* __restrict__ tw,
                 long long batch, float csign) {
  constexpr int R = P::R(0);
  static_assert(P::S == 2 && P::R(1) == R && P::TPF == R && R <= 32 && (R & (R - 1)) == 0 && P::MAP == LT_FAST,
                "shuffle exchange: N = R x R, R lanes per transform");
  int f, lt;
  P::thread_coords(threadIdx.x, f, lt);
  const long long t = (long long)blockIdx.x * P::FPB + f;
  // every lane of a transform group takes part in the shuffles; only valid transforms touch HBM
  const bool valid = t < batch;
  const float2* gi = in + (valid ? t : 0) * P::N;
  float2* go = out + (valid ? t : 0) * P::N;
  float2 v[R];
  sfor<R>([&](auto r_) {
    constexpr int r = decltype(r_)::value;
    const float2 a = valid ? __ldcs(gi + lt + r * R) : make_float2(0.f, 0.f);
    v[r] = make_float2(a.x, csign * a.y);
  });
  Codelet<R>::run(v);
  lane_transpose<R>(v, lt);
  // stage 1 (Ns = R, m = lt): w_N^{lt r}, r = 2^b loaded, the others formed as products
  const float2* tp = tw + (R - 1) + lt;
  float2 w[R];
  sfor<R - 1>([&](auto r_) {
    constexpr int r = decltype(r_)::value + 1;
    constexpr int hb = highbit(r);
    if constexpr (hb == r) w[r] = __ldg(tp + (r - 1) * R);
    else w[r] = cmul(w[hb], w[r - hb]);
    v[r] = cmul(v[r], w[r]);
  });
  Codelet<R>::run(v);
  if (valid)
    sfor<R>([&](auto r_) {
      constexpr int r = decltype(r_)::value;
      __stcs(go + lt + r * R, make_float2(v[r].x, csign * v[r].y));
    });
}

template <class P, int MINB>
static cudaError_t launch_fused_shfl(const float2* in, float2* out, const float2* tw, long long batch, int conj,
                                     cudaStream_t st) {
  const long long grid = (batch + P::FPB - 1) / P::FPB;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  k_fused_shfl<P, MINB><<<(unsigned)grid, P::THREADS, 0, st>>>(in, out, tw, batch, conj ? -1.0f : 1.0f);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- persistent register-pipelined kernel
// LT_FAST direct schedules.  Each CTA loops over tiles of FPB transforms; the stage-0 inputs of
// the CTA's NEXT tile are loaded into registers (plain coalesced loads, the same lanes and
// elements stage 0 consumes) before the current tile's stages run, so every CTA keeps HBM
// reads in flight while it computes instead of issuing them in one burst per tile.
template <class P, int MINB>
__global__ void __launch_bounds__(P::THREADS, MINB)
    k_fused_pipe(const float2* __restrict__ in, float2* __restrict__ out, const float2* __restrict__ tw,
                 long long batch, float csign) {
  static_assert(P::MAP == LT_FAST, "register pipeline: LT_FAST mapping");
  extern __shared__ float2 sm[];
  constexpr int N = P::N, R = P::R(0), NB = N / R, KB = (NB + P::TPF - 1) / P::TPF;
  constexpr bool EXACT = (NB % P::TPF) == 0;
  int f, lt;
  P::thread_coords(threadIdx.x, f, lt);
  const long long ntiles = (batch + P::FPB - 1) / P::FPB;
  float2 pre[KB][R];
  auto fetch = [&](long long t) {
    const long long tr = t * P::FPB + f;
    if (t < ntiles && tr < batch) {
      const float2* gi = in + tr * N;
      sfor<KB>([&](auto k_) {
        constexpr int k = decltype(k_)::value;
        const int j = lt + k * P::TPF;
        if (EXACT || j < NB)
          sfor<R>([&](auto r_) {
            constexpr int r = decltype(r_)::value;
            pre[k][r] = __ldcs(gi + j + r * NB);
          });
      });
    }
  };
  long long t = blockIdx.x;
  fetch(t);
  for (; t < ntiles; t += gridDim.x) {
    const long long tr = t * P::FPB + f;
    const bool fvalid = tr < batch;
    float2 v[KB][R];
    sfor<KB>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      sfor<R>([&](auto r_) {
        constexpr int r = decltype(r_)::value;
        v[k][r] = make_float2(pre[k][r].x, csign * pre[k][r].y);
      });
    });
    fetch(t + gridDim.x);  // next tile's stage-0 inputs: in flight during this tile's stages
    // stage 0 from registers (Ns = 1: no twiddle, outputs j R + r) into the exchange buffer
    sfor<KB>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      const int j = lt + k * P::TPF;
      if (fvalid && (EXACT || j < NB)) {
        Codelet<R>::run(v[k]);
        sfor<R>([&](auto r_) {
          constexpr int r = decltype(r_)::value;
          sm[P::sidx(f, j * R + r)] = v[k][r];
        });
      }
    });
    P::sync();
    float2* go = out + tr * N;
    sfor<P::S - 1>([&](auto s_) {
      constexpr int s = decltype(s_)::value + 1;
      stage<P, s, false, s == P::S - 1>(
          sm, f, lt, fvalid, tw, [&](int, int) { return make_float2(0.f, 0.f); },
          [&](int i, float2 w, int) { __stcs(go + i, make_float2(w.x, csign * w.y)); });
    });
    P::sync();  // the exchange buffer is free for the next tile's stage 0
  }
}

template <class P, int MINB>
static cudaError_t launch_fused_pipe(const float2* in, float2* out, const float2* tw, long long batch, int conj,
                                     cudaStream_t st) {
  auto kern = k_fused_pipe<P, MINB>;
  static PerDevice<KernelSetup> ks_pd;
  const KernelSetup& ks = ks_pd.get([&] { return kernel_setup(kern, P::THREADS, P::SMEM); });
  if (ks.err != cudaSuccess) return ks.err;
  const int grid_max = ks.grid_max;
  const long long ntiles = (batch + P::FPB - 1) / P::FPB;
  if (ntiles == 0) return cudaSuccess;
  const unsigned grid = (unsigned)(ntiles < grid_max ? ntiles : grid_max);
  kern<<<grid, P::THREADS, P::SMEM, st>>>(in, out, tw, batch, conj ? -1.0f : 1.0f);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- persistent TMA-fed kernel
// LT_FAST schedules (S >= 2).  Each CTA loops over tiles of FPB contiguous transforms.
// A tile is brought HBM -> shared by one bulk asynchronous copy (cp.async.bulk, TMA
// engine, completion on an mbarrier) into a linear buffer LIN; stage 0 reads LIN and
// writes the swizzled exchange buffer WORK; as soon as every thread has read LIN, the
// copy of the CTA's next tile is issued, so it streams in while stages 1..S-1 run and
// the last stage stores HBM directly.
template <class P, int MINB>
__global__ void __launch_bounds__(P::THREADS, MINB)
    k_fused_tma(const float2* __restrict__ in, float2* __restrict__ out, const float2* __restrict__ tw,
                long long batch, float csign) {
  static_assert(P::MAP == LT_FAST && P::S >= 2, "TMA kernel: LT_FAST, at least two stages");
  constexpr int N = P::N, FPB = P::FPB;
  constexpr int WORK = ((P::SS * FPB) + 1) & ~1;  // keep LIN 16-byte aligned
  extern __shared__ __align__(128) float2 sm[];
  float2* work = sm;
  float2* lin = sm + WORK;
  __shared__ __align__(8) uint64_t bar;
  int f, lt;
  P::thread_coords(threadIdx.x, f, lt);
  const long long ntiles = (batch + FPB - 1) / FPB;
  auto tile_nf = [&](long long t) {
    const long long rem = batch - t * FPB;
    return rem < FPB ? (int)rem : FPB;
  };
  auto tile_tma = [&](long long t) { return ((long long)tile_nf(t) * N * 8) % 16 == 0; };
  auto issue = [&](long long t) {
    const uint32_t bytes = (uint32_t)tile_nf(t) * N * 8u;
    mbar_arrive_expect_tx(&bar, bytes);
    bulk_g2s(lin, in + t * FPB * (long long)N, bytes, &bar);
  };
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  long long t = blockIdx.x;
  uint32_t phase = 0;
  if (threadIdx.x == 0 && t < ntiles && tile_tma(t)) issue(t);
  for (; t < ntiles; t += gridDim.x) {
    const int nf = tile_nf(t);
    const bool fvalid = f < nf;
    if (tile_tma(t)) {
      mbar_wait(&bar, phase);
      phase ^= 1;
    } else {  // ragged odd-length tail tile: plain copy
      const float2* g = in + t * FPB * (long long)N;
      for (int e = threadIdx.x; e < nf * N; e += P::THREADS) lin[e] = g[e];
    }
    __syncthreads();  // WORK free (previous tile's last stage done), LIN visible
    float2* go = out + t * FPB * (long long)N + (long long)f * N;
    const float2* gl = lin + f * N;
    auto gstore = [&](int i, float2 v, int) { __stcs(go + i, make_float2(v.x, csign * v.y)); };
    stage<P, 0, true, false>(
        work, f, lt, fvalid, tw,
        [&](int i, int) {
          const float2 a = gl[i];
          return make_float2(a.x, csign * a.y);
        },
        gstore);
    fence_proxy_async_smem();
    __syncthreads();  // every thread has read LIN
    if (threadIdx.x == 0) {
      const long long tn = t + gridDim.x;
      if (tn < ntiles && tile_tma(tn)) issue(tn);
    }
    sfor<P::S - 1>([&](auto s_) {
      constexpr int s = decltype(s_)::value + 1;
      stage<P, s, false, s == P::S - 1>(work, f, lt, fvalid, tw, [&](int, int) { return make_float2(0.f, 0.f); },
                                        gstore);
    });
  }
}

template <class P, int MINB>
static cudaError_t launch_fused_tma(const float2* in, float2* out, const float2* tw, long long batch, int conj,
                                    cudaStream_t st) {
  auto kern = k_fused_tma<P, MINB>;
  constexpr size_t smem = (size_t)((((P::SS * P::FPB) + 1) & ~1) + P::N * P::FPB) * sizeof(float2);
  static PerDevice<KernelSetup> ks_pd;
  const KernelSetup& ks = ks_pd.get([&] { return kernel_setup(kern, P::THREADS, smem); });
  if (ks.err != cudaSuccess) return ks.err;
  const int grid_max = ks.grid_max;
  const long long ntiles = (batch + P::FPB - 1) / P::FPB;
  if (ntiles == 0) return cudaSuccess;
  const unsigned grid = (unsigned)(ntiles < grid_max ? ntiles : grid_max);
  kern<<<grid, P::THREADS, smem, st>>>(in, out, tw, batch, conj ? -1.0f : 1.0f);
  return cudaGetLastError();
}

}  // namespace fftc
