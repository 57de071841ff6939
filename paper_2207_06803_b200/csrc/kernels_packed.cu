// kernels_packed.cu -- compiled single-pass schedules whose register codelets use sm_100's
// paired FP32 arithmetic (FFTC_PACKED, codelets.cuh: FADD2 / FMUL2 / FFMA2 on (re, im) pairs)
// (product path).  Only the sizes where it measured faster through bench.py on B200 (DESIGN §9:
// 105 -6 %, 210 -2 %, 1000 -3 %, 3125 -5 %, 128 -5 %; tools/tune.py: 1000 with 100x2 threads
// and 2048 another -1 %); their rows come first in the registry,
// so they are the defaults, and the scalar rows stay as candidates.  Each .cu is its own device
// module (no -rdc), so the packed codelets never mix with the scalar ones; TAG = 1 keeps the
// kernel symbols distinct from the scalar schedules of the same shape.
#define FFTC_PACKED 1
#include "kernels_common.cuh"

namespace fftc {

#define FFTC_ENTRY_PK(NAME, N, RAD, TPF, FPB, MAP, DIRECT, MINB, ...)                                  \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, DIRECT,                                             \
   Sched<N, RAD, TPF, FPB, MAP, 0, LAY_AUTO, 1>::SMEM,                                                \
   &launch_fused_batch<Sched<N, RAD, TPF, FPB, MAP, 0, LAY_AUTO, 1>, DIRECT, MINB>, NAME}

#define FFTC_ENTRY_PK_OPT(NAME, N, RAD, TPF, FPB, MINB, OPT, ...)                                     \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, true,                                               \
   Sched<N, RAD, TPF, FPB, LT_FAST, 0, LAY_AUTO, 1, OPT>::SMEM,                                        \
   &launch_fused_batch<Sched<N, RAD, TPF, FPB, LT_FAST, 0, LAY_AUTO, 1, OPT>, true, MINB>, NAME}

extern const FusedEntry kTable_packed[];
extern const int kCount_packed;
const FusedEntry kTable_packed[] = {
    FFTC_ENTRY_PK("n128_r8x16_t16x4d_pk", 128, Rad_8x16, 16, 4, LT_FAST, true, 16, 8, 16),
    FFTC_ENTRY_PK("n105_r7x15_t8x16d_pk", 105, Rad_7x15, 8, 16, LT_FAST, true, 8, 7, 15),
    FFTC_ENTRY_PK("n210_r14x15_t15x8d_pk", 210, Rad_14x15, 15, 8, LT_FAST, true, 8, 14, 15),
    FFTC_ENTRY_PK("n1000_r10x10x10_t100x2_pk", 1000, Rad_10x10x10, 100, 2, LT_FAST, true, 4, 10, 10, 10),
    FFTC_ENTRY_PK("n3125_r25x5x25_t128x1_pk", 3125, Rad_25x5x25, 128, 1, LT_FAST, true, 4, 25, 5, 25),
    // default for 2048: paired FP32 + stage-0 loads with L1::no_allocate (162.9 vs 164.3 us)
    FFTC_ENTRY_PK_OPT("n2048_r16x16x8_t128x1_pk_na", 2048, Rad_16x16x8, 128, 1, 4, OPT_LD_NA, 16, 16, 8),
    FFTC_ENTRY_PK("n2048_r16x16x8_t128x1_pk", 2048, Rad_16x16x8, 128, 1, LT_FAST, true, 4, 16, 16, 8),
};
const int kCount_packed = (int)(sizeof(kTable_packed) / sizeof(kTable_packed[0]));

// paired-FP32 candidates for the other schedules (registered after every scalar table, so
// they never become defaults; tools/tune.py / FFTC_KERNEL select them)
extern const FusedEntry kTable_packed_cand[];
extern const int kCount_packed_cand;
const FusedEntry kTable_packed_cand[] = {
    FFTC_ENTRY_PK_OPT("n3125_r25x5x25_t128x1_pk_na", 3125, Rad_25x5x25, 128, 1, 4, OPT_LD_NA, 25, 5, 25),
    FFTC_ENTRY_PK_OPT("n1000_r10x10x10_t100x2_pk_na", 1000, Rad_10x10x10, 100, 2, 4, OPT_LD_NA, 10, 10, 10),
    FFTC_ENTRY_PK_OPT("n2187_r27x9x9_t81x2_pk_sh", 2187, Rad_27x9x9, 81, 2, 3, OPT_TW_SHARE, 27, 9, 9),
    FFTC_ENTRY_PK_OPT("n3125_r25x5x25_t125x2_pk_sh", 3125, Rad_25x5x25, 125, 2, 3, OPT_TW_SHARE, 25, 5, 25),
    FFTC_ENTRY_PK_OPT("n1000_r10x10x10_t50x2_pk_vsh", 1000, Rad_10x10x10, 50, 2, 6, OPT_VEC_IO | OPT_TW_SHARE, 10, 10,
                      10),
    FFTC_ENTRY_PK_OPT("n1000_r10x10x10_t100x2_pk_v", 1000, Rad_10x10x10, 100, 2, 4, OPT_VEC_IO, 10, 10, 10),
    FFTC_ENTRY_PK_OPT("n4096_r16x16x16_t128x1_pk_vsh", 4096, Rad_16x16x16, 128, 1, 4, OPT_VEC_IO | OPT_TW_SHARE, 16,
                      16, 16),
    FFTC_ENTRY_PK("n2187_r27x9x9_t128x1_pk", 2187, Rad_27x9x9, 128, 1, LT_FAST, true, 4, 27, 9, 9),
    FFTC_ENTRY_PK("n2187_r27x9x9_t81x2_pk", 2187, Rad_27x9x9, 81, 2, LT_FAST, true, 3, 27, 9, 9),
    FFTC_ENTRY_PK("n2187_r9x9x27_t81x2_pk", 2187, Rad_9x9x27, 81, 2, LT_FAST, true, 3, 9, 9, 27),
    FFTC_ENTRY_PK("n2187_r3x27x27_t81x1_pk", 2187, Rad_3x27x27, 81, 1, LT_FAST, true, 6, 3, 27, 27),
    FFTC_ENTRY_PK("n1000_r10x10x10_t50x2_pk", 1000, Rad_10x10x10, 50, 2, LT_FAST, true, 6, 10, 10, 10),
    FFTC_ENTRY_PK("n1000_r10x10x10_t50x4_pk", 1000, Rad_10x10x10, 50, 4, LT_FAST, true, 3, 10, 10, 10),
    FFTC_ENTRY_PK("n3125_r25x5x25_t125x2_pk", 3125, Rad_25x5x25, 125, 2, LT_FAST, true, 3, 25, 5, 25),
    FFTC_ENTRY_PK("n3125_r5x25x25_t125x2_pk", 3125, Rad_5x25x25, 125, 2, LT_FAST, true, 3, 5, 25, 25),
    FFTC_ENTRY_PK("n60_r4x15_t4x16d_pk", 60, Rad_4x15, 4, 16, LT_FAST, true, 16, 4, 15),
    FFTC_ENTRY_PK("n4096_r16x16x16_t256x1_pk", 4096, Rad_16x16x16, 256, 1, LT_FAST, true, 3, 16, 16, 16),
};
const int kCount_packed_cand = (int)(sizeof(kTable_packed_cand) / sizeof(kTable_packed_cand[0]));

}  // namespace fftc
