// kernels_batch.cu -- compiled single-pass schedules for the BASELINE.json sizes.
//
// Each row: N, radix list (R_0 = leaf DFT, innermost level of Eq. 2), thread
// mapping, threads per transform, transforms per CTA.  See DESIGN.md §6 for the
// per-size choice (register budget, shared-memory exchanges, coalescing).
#include "fused.cuh"
#include "registry.h"

namespace fftc {

#define FFTC_ENTRY(NAME, N, RAD, TPF, FPB, MAP, DIRECT, MINB, ...)                                  \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, DIRECT,                                        \
   Sched<N, RAD, TPF, FPB, MAP>::SMEM, &launch_fused_batch<Sched<N, RAD, TPF, FPB, MAP>, DIRECT, MINB>, \
   NAME}

using Rad_10x10x10 = Radices<10, 10, 10>;
using Rad_14x15 = Radices<14, 15>;
using Rad_16 = Radices<16>;
using Rad_16x16 = Radices<16, 16>;
using Rad_16x16x16 = Radices<16, 16, 16>;
using Rad_16x32 = Radices<16, 32>;
using Rad_3x5x7 = Radices<3, 5, 7>;
using Rad_32x32 = Radices<32, 32>;
using Rad_4x3x5 = Radices<4, 3, 5>;
using Rad_4x8 = Radices<4, 8>;
using Rad_5x25x25 = Radices<5, 25, 25>;
using Rad_8 = Radices<8>;
using Rad_8x16 = Radices<8, 16>;
using Rad_8x16x16 = Radices<8, 16, 16>;
using Rad_8x8 = Radices<8, 8>;
using Rad_9x9x27 = Radices<9, 9, 27>;

static const FusedEntry kTable[] = {
    // tiny N: one thread holds a whole transform; I/O staged (128-bit, contiguous)
    FFTC_ENTRY("n8_r8_t1x128", 8, Rad_8, 1, 128, F_FAST, false, 4, 8),
    FFTC_ENTRY("n16_r16_t1x128", 16, Rad_16, 1, 128, F_FAST, false, 4, 16),
    FFTC_ENTRY("n32_r4x8_t4x64", 32, Rad_4x8, 4, 64, F_FAST, false, 4, 4, 8),
    FFTC_ENTRY("n64_r8x8_t8x32", 64, Rad_8x8, 8, 32, F_FAST, false, 4, 8, 8),
    FFTC_ENTRY("n128_r8x16_t8x32", 128, Rad_8x16, 8, 32, F_FAST, false, 3, 8, 16),
    // mixed radix (BASELINE.json config 3)
    FFTC_ENTRY("n60_r4x3x5_t4x64", 60, Rad_4x3x5, 4, 64, F_FAST, false, 4, 4, 3, 5),
    FFTC_ENTRY("n105_r3x5x7_t8x32", 105, Rad_3x5x7, 8, 32, F_FAST, false, 4, 3, 5, 7),
    FFTC_ENTRY("n210_r14x15_t15x16", 210, Rad_14x15, 15, 16, F_FAST, false, 3, 14, 15),
    FFTC_ENTRY("n1000_r10x10x10_t100x2", 1000, Rad_10x10x10, 100, 2, LT_FAST, true, 4, 10, 10, 10),
    FFTC_ENTRY("n2187_r9x9x27_t81x2", 2187, Rad_9x9x27, 81, 2, LT_FAST, true, 3, 9, 9, 27),
    FFTC_ENTRY("n3125_r5x25x25_t125x2", 3125, Rad_5x25x25, 125, 2, LT_FAST, true, 3, 5, 25, 25),
    // large power-of-two N: lanes walk one transform, HBM read/written by the first/last stage
    FFTC_ENTRY("n256_r16x16_t16x16", 256, Rad_16x16, 16, 16, LT_FAST, true, 3, 16, 16),
    FFTC_ENTRY("n512_r16x32_t16x16", 512, Rad_16x32, 16, 16, LT_FAST, true, 2, 16, 32),
    FFTC_ENTRY("n1024_r32x32_t32x8", 1024, Rad_32x32, 32, 8, LT_FAST, true, 2, 32, 32),
    FFTC_ENTRY("n2048_r8x16x16_t128x2", 2048, Rad_8x16x16, 128, 2, LT_FAST, true, 3, 8, 16, 16),
    FFTC_ENTRY("n4096_r16x16x16_t256x1", 4096, Rad_16x16x16, 256, 1, LT_FAST, true, 3, 16, 16, 16),
};

const FusedEntry* find_fused(int N) {
  for (const auto& e : kTable)
    if (e.N == N) return &e;
  return nullptr;
}
int fused_count() { return (int)(sizeof(kTable) / sizeof(kTable[0])); }
const FusedEntry* fused_at(int i) { return (i >= 0 && i < fused_count()) ? &kTable[i] : nullptr; }

}  // namespace fftc
