// kernels_small.cu -- compiled single-pass schedules, small sizes (product path).
// Row: name, N, radix list (R_0 = leaf DFT, innermost level of Eq. 2), threads per
// transform, transforms per CTA, mapping, direct HBM I/O, min CTAs/SM, radices.  The first
// row for an N is the planner's default; the others are candidates (tools/tune.py).
#include "kernels_common.cuh"

namespace fftc {

extern const FusedEntry kTable_small[];
extern const int kCount_small;
const FusedEntry kTable_small[] = {
    FFTC_ENTRY("n8_r8_t1x128", 8, Rad_8, 1, 128, F_FAST, false, 4, 8),
    FFTC_ENTRY("n16_r16_t1x128", 16, Rad_16, 1, 128, F_FAST, false, 4, 16),
    FFTC_ENTRY("n32_r32_t1x128", 32, Rad_32, 1, 128, F_FAST, false, 2, 32),
    FFTC_ENTRY("n32_r4x8_t4x64", 32, Rad_4x8, 4, 64, F_FAST, false, 4, 4, 8),
    // default: the stage exchange as an 8 x 8 lane transpose by warp shuffles (no shared memory);
    // measured on B200 against the shared-memory exchange (profiles/r02b/shfl64.jsonl): 167.6 vs 169.8 us
    FFTC_SHFL("n64_r8x8_t8x8_shfl", 64, Rad_8x8, 8, 8, 16, 8, 8),
    FFTC_ENTRY("n64_r8x8_t8x8d", 64, Rad_8x8, 8, 8, LT_FAST, true, 16, 8, 8),
    FFTC_ENTRY("n64_r8x8_t8x32", 64, Rad_8x8, 8, 32, F_FAST, false, 4, 8, 8),
    FFTC_ENTRY("n64_r4x16_t4x64", 64, Rad_4x16, 4, 64, F_FAST, false, 4, 4, 16),
    FFTC_ENTRY("n64_r16x4_t4x64", 64, Rad_16x4, 4, 64, F_FAST, false, 4, 16, 4),
    FFTC_ENTRY("n128_r8x16_t16x4d", 128, Rad_8x16, 16, 4, LT_FAST, true, 16, 8, 16),
    FFTC_ENTRY("n128_r8x16_t8x32", 128, Rad_8x16, 8, 32, F_FAST, false, 3, 8, 16),
    FFTC_ENTRY("n128_r16x8_t8x32", 128, Rad_16x8, 8, 32, F_FAST, false, 3, 16, 8),
    FFTC_ENTRY("n128_r8x16_t8x16", 128, Rad_8x16, 8, 16, F_FAST, false, 6, 8, 16),
    FFTC_ENTRY("n128_r8x16_t16x16d", 128, Rad_8x16, 16, 16, LT_FAST, true, 4, 8, 16),
    FFTC_ENTRY("n64_r8x8_t8x16", 64, Rad_8x8, 8, 16, F_FAST, false, 8, 8, 8),
    FFTC_SHFL("n64_r8x8_t8x16_shfl", 64, Rad_8x8, 8, 16, 8, 8, 8),
    FFTC_ENTRY("n128_r16x8_t16x16d", 128, Rad_16x8, 16, 16, LT_FAST, true, 4, 16, 8),
    FFTC_ENTRY("n128_r8x16_t16x8d", 128, Rad_8x16, 16, 8, LT_FAST, true, 8, 8, 16),
    FFTC_ENTRY("n128_r8x16_t8x8", 128, Rad_8x16, 8, 8, F_FAST, false, 8, 8, 16),
    FFTC_ENTRY("n64_r8x8_t8x8", 64, Rad_8x8, 8, 8, F_FAST, false, 16, 8, 8),
    FFTC_ENTRY("n128_r16x8_t16x8d", 128, Rad_16x8, 16, 8, LT_FAST, true, 8, 16, 8),
};
const int kCount_small = (int)(sizeof(kTable_small) / sizeof(kTable_small[0]));

}  // namespace fftc
