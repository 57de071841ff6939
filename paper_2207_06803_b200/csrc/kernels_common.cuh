// kernels_common.cuh -- shared macros/aliases of the compiled single-pass schedules (product path).
#pragma once
#include "fused.cuh"
#include "registry.h"

namespace fftc {

#define FFTC_ENTRY(NAME, N, RAD, TPF, FPB, MAP, DIRECT, MINB, ...)                                  \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, DIRECT,                                        \
   Sched<N, RAD, TPF, FPB, MAP>::SMEM, &launch_fused_batch<Sched<N, RAD, TPF, FPB, MAP>, DIRECT, MINB>, \
   NAME}
// LT_FAST with the row padded to a multiple of 16 so the XOR swizzle applies to any N
#define FFTC_ENTRY_PAD(NAME, N, RAD, TPF, FPB, PAD, MINB, ...)                                  \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, true,                                        \
   Sched<N, RAD, TPF, FPB, LT_FAST, PAD>::SMEM, &launch_fused_batch<Sched<N, RAD, TPF, FPB, LT_FAST, PAD>, true, MINB>, \
   NAME}
// LT_FAST direct schedule with SchedOpt options (fused.cuh: OPT_TW_LOAD, OPT_VEC_IO, OPT_TW_SHARE)
#define FFTC_ENTRY_OPT(NAME, N, RAD, TPF, FPB, MINB, OPT, ...)                                     \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, true,                                          \
   Sched<N, RAD, TPF, FPB, LT_FAST, 0, LAY_AUTO, 0, OPT>::SMEM,                                   \
   &launch_fused_batch<Sched<N, RAD, TPF, FPB, LT_FAST, 0, LAY_AUTO, 0, OPT>, true, MINB>, NAME}
// LT_FAST direct schedule with the padded shared layout (LAY_PAD16) and SchedOpt options
#define FFTC_ENTRY_P16(NAME, N, RAD, TPF, FPB, MINB, OPT, ...)                                     \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, true,                                          \
   Sched<N, RAD, TPF, FPB, LT_FAST, 0, LAY_PAD16, 0, OPT>::SMEM,                                  \
   &launch_fused_batch<Sched<N, RAD, TPF, FPB, LT_FAST, 0, LAY_PAD16, 0, OPT>, true, MINB>, NAME}
// warp-shuffle exchange variant (N = R x R, TPF = R; fused.cuh k_fused_shfl), no shared memory
#define FFTC_SHFL(NAME, N, RAD, TPF, FPB, MINB, ...)                                               \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, true, 0,                                        \
   &launch_fused_shfl<Sched<N, RAD, TPF, FPB, LT_FAST>, MINB>, NAME}
// persistent, TMA-fed variant (LT_FAST schedules)
#define FFTC_TMA(NAME, N, RAD, TPF, FPB, MINB, ...)                                               \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, 2, Sched<N, RAD, TPF, FPB, LT_FAST>::SMEM * 2,    \
   &launch_fused_tma<Sched<N, RAD, TPF, FPB, LT_FAST>, MINB>, NAME}

// persistent, register-pipelined variant (LT_FAST direct schedules)
#define FFTC_PIPE(NAME, N, RAD, TPF, FPB, MINB, ...)                                              \
  {N, RAD::S, {__VA_ARGS__}, TPF, FPB, TPF * FPB, 3, Sched<N, RAD, TPF, FPB, LT_FAST>::SMEM,      \
   &launch_fused_pipe<Sched<N, RAD, TPF, FPB, LT_FAST>, MINB>, NAME}

using Rad_8 = Radices<8>;
using Rad_16 = Radices<16>;
using Rad_32 = Radices<32>;
using Rad_4x8 = Radices<4, 8>;
using Rad_8x4 = Radices<8, 4>;
using Rad_8x8 = Radices<8, 8>;
using Rad_4x16 = Radices<4, 16>;
using Rad_16x4 = Radices<16, 4>;
using Rad_8x16 = Radices<8, 16>;
using Rad_16x8 = Radices<16, 8>;
using Rad_4x32 = Radices<4, 32>;
using Rad_16x16 = Radices<16, 16>;
using Rad_16x32 = Radices<16, 32>;
using Rad_32x16 = Radices<32, 16>;
using Rad_32x32 = Radices<32, 32>;
using Rad_8x16x16 = Radices<8, 16, 16>;
using Rad_16x16x8 = Radices<16, 16, 8>;
using Rad_16x16x16 = Radices<16, 16, 16>;
using Rad_4x3x5 = Radices<4, 3, 5>;
using Rad_4x15 = Radices<4, 15>;
using Rad_3x5x7 = Radices<3, 5, 7>;
using Rad_7x15 = Radices<7, 15>;
using Rad_14x15 = Radices<14, 15>;
using Rad_10x10x10 = Radices<10, 10, 10>;
using Rad_9x9x27 = Radices<9, 9, 27>;
using Rad_5x25x25 = Radices<5, 25, 25>;

using Rad_16x8x16 = Radices<16, 8, 16>;
using Rad_16x32x8 = Radices<16, 32, 8>;
using Rad_8x32x16 = Radices<8, 32, 16>;
using Rad_8x8x8x8 = Radices<8, 8, 8, 8>;
using Rad_15x14 = Radices<15, 14>;
using Rad_3x27x27 = Radices<3, 27, 27>;
using Rad_25x25x5 = Radices<25, 25, 5>;
using Rad_6x35 = Radices<6, 35>;
using Rad_27x9x9 = Radices<27, 9, 9>;
using Rad_9x27x9 = Radices<9, 27, 9>;
using Rad_15x4 = Radices<15, 4>;
using Rad_15x7 = Radices<15, 7>;
using Rad_7x30 = Radices<7, 30>;
using Rad_25x40 = Radices<25, 40>;
using Rad_40x25 = Radices<40, 25>;
using Rad_25x5x25 = Radices<25, 5, 25>;

}  // namespace fftc
