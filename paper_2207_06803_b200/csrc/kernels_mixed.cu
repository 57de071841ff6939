// kernels_mixed.cu -- compiled single-pass schedules, mixed sizes (product path).
// Row: name, N, radix list (R_0 = leaf DFT, innermost level of Eq. 2), threads per
// transform, transforms per CTA, mapping, direct HBM I/O, min CTAs/SM, radices.  The first
// row for an N is the planner's default; the others are candidates (tools/tune.py).
#include "kernels_common.cuh"

namespace fftc {

extern const FusedEntry kTable_mixed[];
extern const int kCount_mixed;
const FusedEntry kTable_mixed[] = {
    // default: staged I/O (interleaved A/B on one box: 172.8 vs 179.6 us for direct I/O,
    // profiles/r02b/defaults_ab.jsonl)
    FFTC_ENTRY("n60_r4x15_t4x16", 60, Rad_4x15, 4, 16, F_FAST, false, 16, 4, 15),
    FFTC_ENTRY("n60_r4x15_t4x16d", 60, Rad_4x15, 4, 16, LT_FAST, true, 16, 4, 15),
    FFTC_ENTRY("n60_r4x3x5_t4x64", 60, Rad_4x3x5, 4, 64, F_FAST, false, 4, 4, 3, 5),
    FFTC_ENTRY("n60_r4x15_t4x64", 60, Rad_4x15, 4, 64, F_FAST, false, 4, 4, 15),
    FFTC_ENTRY("n105_r7x15_t8x16d", 105, Rad_7x15, 8, 16, LT_FAST, true, 8, 7, 15),
    FFTC_ENTRY("n105_r7x15_t8x16", 105, Rad_7x15, 8, 16, F_FAST, false, 8, 7, 15),
    FFTC_ENTRY("n105_r3x5x7_t8x32", 105, Rad_3x5x7, 8, 32, F_FAST, false, 4, 3, 5, 7),
    FFTC_ENTRY("n105_r7x15_t8x32", 105, Rad_7x15, 8, 32, F_FAST, false, 4, 7, 15),
    FFTC_ENTRY("n210_r14x15_t15x8d", 210, Rad_14x15, 15, 8, LT_FAST, true, 8, 14, 15),
    FFTC_ENTRY("n210_r7x30_t8x16", 210, Rad_7x30, 8, 16, F_FAST, false, 4, 7, 30),
    FFTC_ENTRY("n210_r14x15_t15x16", 210, Rad_14x15, 15, 16, F_FAST, false, 3, 14, 15),
    FFTC_ENTRY("n1000_r10x10x10_t50x2", 1000, Rad_10x10x10, 50, 2, LT_FAST, true, 6, 10, 10, 10),
    FFTC_ENTRY("n1000_r10x10x10_t100x2", 1000, Rad_10x10x10, 100, 2, LT_FAST, true, 4, 10, 10, 10),
    FFTC_ENTRY("n1000_r10x10x10_t50x4", 1000, Rad_10x10x10, 50, 4, LT_FAST, true, 3, 10, 10, 10),
    FFTC_ENTRY("n2187_r27x9x9_t128x1", 2187, Rad_27x9x9, 128, 1, LT_FAST, true, 4, 27, 9, 9),
    FFTC_ENTRY("n2187_r9x9x27_t81x2", 2187, Rad_9x9x27, 81, 2, LT_FAST, true, 3, 9, 9, 27),
    FFTC_ENTRY("n3125_r25x5x25_t128x1", 3125, Rad_25x5x25, 128, 1, LT_FAST, true, 4, 25, 5, 25),
    FFTC_ENTRY("n3125_r25x5x25_t125x2", 3125, Rad_25x5x25, 125, 2, LT_FAST, true, 3, 25, 5, 25),
    FFTC_ENTRY("n3125_r5x25x25_t125x2", 3125, Rad_5x25x25, 125, 2, LT_FAST, true, 3, 5, 25, 25),
    FFTC_ENTRY("n60_r4x15_t4x32", 60, Rad_4x15, 4, 32, F_FAST, false, 8, 4, 15),
    FFTC_ENTRY("n1000_r25x40_t40x4", 1000, Rad_25x40, 40, 4, LT_FAST, true, 4, 25, 40),
    FFTC_ENTRY("n210_r15x14_t15x8", 210, Rad_15x14, 15, 8, F_FAST, false, 8, 15, 14),
    FFTC_ENTRY("n210_r15x14_t15x16", 210, Rad_15x14, 15, 16, F_FAST, false, 4, 15, 14),
    // round 2: shared stage twiddles (TPF % Ns == 0), paired 128-bit I/O (even N), all twiddles loaded
    FFTC_ENTRY_OPT("n2187_r27x9x9_t128x1_na", 2187, Rad_27x9x9, 128, 1, 4, OPT_LD_NA, 27, 9, 9),
    FFTC_ENTRY_OPT("n3125_r25x5x25_t128x1_na", 3125, Rad_25x5x25, 128, 1, 4, OPT_LD_NA, 25, 5, 25),
    FFTC_ENTRY_OPT("n2187_r27x9x9_t81x2_sh", 2187, Rad_27x9x9, 81, 2, 3, OPT_TW_SHARE, 27, 9, 9),
    FFTC_ENTRY_OPT("n2187_r27x9x9_t81x2_shl", 2187, Rad_27x9x9, 81, 2, 3, OPT_TW_SHARE | OPT_TW_LOAD, 27, 9, 9),
    FFTC_ENTRY_OPT("n2187_r27x9x9_t128x1_l", 2187, Rad_27x9x9, 128, 1, 4, OPT_TW_LOAD, 27, 9, 9),
    FFTC_ENTRY_OPT("n3125_r25x5x25_t125x2_sh", 3125, Rad_25x5x25, 125, 2, 3, OPT_TW_SHARE, 25, 5, 25),
    FFTC_ENTRY_OPT("n1000_r10x10x10_t50x2_vsh", 1000, Rad_10x10x10, 50, 2, 6, OPT_VEC_IO | OPT_TW_SHARE, 10, 10, 10),
    FFTC_ENTRY_OPT("n1000_r10x10x10_t100x2_v", 1000, Rad_10x10x10, 100, 2, 4, OPT_VEC_IO, 10, 10, 10),
    FFTC_ENTRY("n1000_r10x10x10_t100x1", 1000, Rad_10x10x10, 100, 1, LT_FAST, true, 8, 10, 10, 10),
    FFTC_ENTRY("n2187_r3x27x27_t81x1", 2187, Rad_3x27x27, 81, 1, LT_FAST, true, 6, 3, 27, 27),
    FFTC_ENTRY("n3125_r25x25x5_t125x1", 3125, Rad_25x25x5, 125, 1, LT_FAST, true, 5, 25, 25, 5),
    FFTC_ENTRY("n210_r15x14_t15x8d", 210, Rad_15x14, 15, 8, LT_FAST, true, 8, 15, 14),
    FFTC_ENTRY("n1000_r10x10x10_t128x1", 1000, Rad_10x10x10, 128, 1, LT_FAST, true, 6, 10, 10, 10),
    FFTC_ENTRY("n2187_r27x9x9_t81x2", 2187, Rad_27x9x9, 81, 2, LT_FAST, true, 3, 27, 9, 9),
    FFTC_ENTRY("n2187_r9x27x9_t81x2", 2187, Rad_9x27x9, 81, 2, LT_FAST, true, 3, 9, 27, 9),
    FFTC_ENTRY("n2187_r9x9x27_t96x2", 2187, Rad_9x9x27, 96, 2, LT_FAST, true, 3, 9, 9, 27),
    FFTC_ENTRY("n3125_r25x5x25_t128x2", 3125, Rad_25x5x25, 128, 2, LT_FAST, true, 2, 25, 5, 25),
    FFTC_ENTRY("n60_r15x4_t15x8d", 60, Rad_15x4, 15, 8, LT_FAST, true, 12, 15, 4),
    FFTC_ENTRY("n105_r7x15_t15x8d", 105, Rad_7x15, 15, 8, LT_FAST, true, 8, 7, 15),
    FFTC_ENTRY("n105_r15x7_t15x8d", 105, Rad_15x7, 15, 8, LT_FAST, true, 8, 15, 7),
    FFTC_ENTRY_PAD("n1000_r10x10x10_t50x2p", 1000, Rad_10x10x10, 50, 2, 8, 6, 10, 10, 10),
    FFTC_ENTRY_PAD("n1000_r10x10x10_t100x2p", 1000, Rad_10x10x10, 100, 2, 8, 4, 10, 10, 10),
    FFTC_ENTRY_PAD("n2187_r27x9x9_t128x1p", 2187, Rad_27x9x9, 128, 1, 5, 4, 27, 9, 9),
    FFTC_ENTRY_PAD("n3125_r25x5x25_t128x1p", 3125, Rad_25x5x25, 128, 1, 11, 4, 25, 5, 25),
};
const int kCount_mixed = (int)(sizeof(kTable_mixed) / sizeof(kTable_mixed[0]));

}  // namespace fftc
