// kernels_large.cu -- compiled single-pass schedules, large sizes (product path).
// Row: name, N, radix list (R_0 = leaf DFT, innermost level of Eq. 2), threads per
// transform, transforms per CTA, mapping, direct HBM I/O, min CTAs/SM, radices.  The first
// row for an N is the planner's default; the others are candidates (tools/tune.py).
#include "kernels_common.cuh"

namespace fftc {

extern const FusedEntry kTable_large[];
extern const int kCount_large;
const FusedEntry kTable_large[] = {
    FFTC_ENTRY("n2048_r16x16x8_t128x1", 2048, Rad_16x16x8, 128, 1, LT_FAST, true, 6, 16, 16, 8),
    FFTC_ENTRY("n2048_r8x16x16_t128x2", 2048, Rad_8x16x16, 128, 2, LT_FAST, true, 3, 8, 16, 16),
    FFTC_ENTRY("n2048_r16x16x8_t128x2", 2048, Rad_16x16x8, 128, 2, LT_FAST, true, 3, 16, 16, 8),
    FFTC_TMA("n2048_r8x16x16_t128x1_tma", 2048, Rad_8x16x16, 128, 1, 6, 8, 16, 16),
    FFTC_PIPE("n2048_r16x16x8_t128x1_pipe3", 2048, Rad_16x16x8, 128, 1, 3, 16, 16, 8),
    // default: 256 threads, stage-0 loads with L1::no_allocate (interleaved A/B on one box: 179.8 vs
    // 182.6 us for the 128-thread no_allocate kernel and 180.4 for 256 threads with plain loads,
    // profiles/r02b/defaults_ab.jsonl)
    FFTC_ENTRY_OPT("n4096_r16x16x16_t256x1_na", 4096, Rad_16x16x16, 256, 1, 3, OPT_LD_NA, 16, 16, 16),
    FFTC_ENTRY_OPT("n4096_r16x16x16_t128x1_na", 4096, Rad_16x16x16, 128, 1, 4, OPT_LD_NA, 16, 16, 16),
    FFTC_ENTRY("n4096_r16x16x16_t128x1", 4096, Rad_16x16x16, 128, 1, LT_FAST, true, 4, 16, 16, 16),
    FFTC_ENTRY("n4096_r16x16x16_t256x1", 4096, Rad_16x16x16, 256, 1, LT_FAST, true, 3, 16, 16, 16),
    FFTC_TMA("n4096_r16x16x16_t256x1_tma", 4096, Rad_16x16x16, 256, 1, 3, 16, 16, 16),
    FFTC_ENTRY("n4096_r16x16x16_t128x1m6", 4096, Rad_16x16x16, 128, 1, LT_FAST, true, 5, 16, 16, 16),
    FFTC_ENTRY("n4096_r16x16x16_t256x1m2", 4096, Rad_16x16x16, 256, 1, LT_FAST, true, 2, 16, 16, 16),
    FFTC_ENTRY("n4096_r16x16x16_t128x1m4", 4096, Rad_16x16x16, 128, 1, LT_FAST, true, 4, 16, 16, 16),
    FFTC_ENTRY("n4096_r16x16x16_t128x1m3", 4096, Rad_16x16x16, 128, 1, LT_FAST, true, 3, 16, 16, 16),
    // round 2: shared stage-1 twiddles (TPF % Ns == 0), paired 128-bit HBM I/O, all twiddles loaded
    FFTC_ENTRY_OPT("n4096_r16x16x16_t128x1_sh", 4096, Rad_16x16x16, 128, 1, 4, OPT_TW_SHARE, 16, 16, 16),
    FFTC_ENTRY_OPT("n4096_r16x16x16_t128x1_v", 4096, Rad_16x16x16, 128, 1, 4, OPT_VEC_IO, 16, 16, 16),
    FFTC_ENTRY_OPT("n4096_r16x16x16_t128x1_vsh", 4096, Rad_16x16x16, 128, 1, 4, OPT_VEC_IO | OPT_TW_SHARE, 16, 16,
                   16),
    FFTC_ENTRY_OPT("n4096_r16x16x16_t128x1_vshl", 4096, Rad_16x16x16, 128, 1, 4,
                   OPT_VEC_IO | OPT_TW_SHARE | OPT_TW_LOAD, 16, 16, 16),
    FFTC_ENTRY_OPT("n4096_r16x16x16_t128x1_l", 4096, Rad_16x16x16, 128, 1, 4, OPT_TW_LOAD, 16, 16, 16),
    FFTC_ENTRY_P16("n4096_r16x16x16_t128x1_p16", 4096, Rad_16x16x16, 128, 1, 4, 0, 16, 16, 16),
    FFTC_ENTRY_P16("n4096_r16x16x16_t128x1_p16sh", 4096, Rad_16x16x16, 128, 1, 4, OPT_TW_SHARE, 16, 16, 16),
    FFTC_ENTRY_P16("n4096_r16x16x16_t256x1_p16", 4096, Rad_16x16x16, 256, 1, 3, 0, 16, 16, 16),
    FFTC_ENTRY_P16("n4096_r16x16x16_t128x1_p16m5", 4096, Rad_16x16x16, 128, 1, 5, 0, 16, 16, 16),
    FFTC_ENTRY_P16("n2048_r16x16x8_t128x1_p16", 2048, Rad_16x16x8, 128, 1, 6, 0, 16, 16, 8),
    FFTC_ENTRY_OPT("n2048_r16x16x8_t128x1_vsh", 2048, Rad_16x16x8, 128, 1, 6, OPT_VEC_IO | OPT_TW_SHARE, 16, 16, 8),
    // register-pipelined persistent candidate (measured 189.8 us vs 183.5 for the default)
    FFTC_PIPE("n4096_r16x16x16_t256x1_pipe2", 4096, Rad_16x16x16, 256, 1, 2, 16, 16, 16),
};
const int kCount_large = (int)(sizeof(kTable_large) / sizeof(kTable_large[0]));

}  // namespace fftc
