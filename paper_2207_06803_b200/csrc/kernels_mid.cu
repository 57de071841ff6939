// kernels_mid.cu -- compiled single-pass schedules, mid sizes (product path).
// Row: name, N, radix list (R_0 = leaf DFT, innermost level of Eq. 2), threads per
// transform, transforms per CTA, mapping, direct HBM I/O, min CTAs/SM, radices.  The first
// row for an N is the planner's default; the others are candidates (tools/tune.py).
#include "kernels_common.cuh"

namespace fftc {

extern const FusedEntry kTable_mid[];
extern const int kCount_mid;
const FusedEntry kTable_mid[] = {
    FFTC_ENTRY("n256_r16x16_t16x8", 256, Rad_16x16, 16, 8, LT_FAST, true, 8, 16, 16),
    FFTC_ENTRY("n256_r16x16_t16x16", 256, Rad_16x16, 16, 16, LT_FAST, true, 3, 16, 16),
    FFTC_TMA("n256_r16x16_t16x16_tma", 256, Rad_16x16, 16, 16, 3, 16, 16),
    FFTC_ENTRY("n512_r32x16_t16x8", 512, Rad_32x16, 16, 8, LT_FAST, true, 4, 32, 16),
    FFTC_ENTRY("n512_r16x32_t16x16", 512, Rad_16x32, 16, 16, LT_FAST, true, 2, 16, 32),
    FFTC_ENTRY("n512_r32x16_t16x16", 512, Rad_32x16, 16, 16, LT_FAST, true, 2, 32, 16),
    FFTC_ENTRY("n1024_r32x32_t32x4", 1024, Rad_32x32, 32, 4, LT_FAST, true, 4, 32, 32),
    FFTC_ENTRY("n1024_r32x32_t32x8", 1024, Rad_32x32, 32, 8, LT_FAST, true, 2, 32, 32),
    FFTC_ENTRY("n512_r32x16_t16x4", 512, Rad_32x16, 16, 4, LT_FAST, true, 8, 32, 16),
    FFTC_ENTRY("n1024_r32x32_t32x2", 1024, Rad_32x32, 32, 2, LT_FAST, true, 8, 32, 32),
    FFTC_SHFL("n256_r16x16_t16x8_shfl", 256, Rad_16x16, 16, 8, 8, 16, 16),
    FFTC_SHFL("n256_r16x16_t16x16_shfl", 256, Rad_16x16, 16, 16, 4, 16, 16),
    FFTC_SHFL("n1024_r32x32_t32x4_shfl", 1024, Rad_32x32, 32, 4, 4, 32, 32),
    FFTC_ENTRY_P16("n1024_r32x32_t32x4_p16", 1024, Rad_32x32, 32, 4, 4, 0, 32, 32),
    FFTC_ENTRY_P16("n512_r32x16_t16x8_p16", 512, Rad_32x16, 16, 8, 4, 0, 32, 16),
    FFTC_ENTRY_P16("n256_r16x16_t16x8_p16", 256, Rad_16x16, 16, 8, 8, 0, 16, 16),
};
const int kCount_mid = (int)(sizeof(kTable_mid) / sizeof(kTable_mid[0]));

}  // namespace fftc
