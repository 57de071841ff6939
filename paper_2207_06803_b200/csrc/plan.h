// plan.h -- the opaque fftc_plan (product path, host side).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fourstep.h"
#include "gpass.h"
#include "jit.h"
#include "c16.h"
#include "direct_tc.h"
#include "l2pass.h"
#include "passes.h"
#include "registry.h"

namespace fftc {

enum PlanKind : int { KIND_COPY = 0, KIND_FUSED = 1, KIND_GENERIC = 2, KIND_FOURSTEP = 3, KIND_DIST = 4, KIND_PASSES = 5, KIND_L2 = 6, KIND_GPASS = 7, KIND_JIT = 8, KIND_DIRECT = 9,
                     KIND_CLUSTER = 10 };

struct DistState;  // dist.cu

struct HostStage {  // fftc_execute_host pipeline buffers
  static constexpr int kDepth = 4;  // max streams / staging slots
  int depth = 3;                     // used (FFTC_HOST_DEPTH)
  int64_t chunk = 0;  // transforms per chunk
  float2* d_in[kDepth] = {};
  float2* d_out[kDepth] = {};
  float2* d_work[kDepth] = {};
  cudaStream_t st[kDepth] = {};
};

}  // namespace fftc

struct fftc_plan {
  int64_t N = 0, batch = 0;
  int sign = -1;
  int device = 0;
  int kind = fftc::KIND_COPY;
  // single pass
  const fftc::FusedEntry* fe = nullptr;
  fftc::GenericSched gs{};
  float2* d_tw = nullptr;  // stage twiddles for N (single pass) or for M (four-step pass 1)
  // four-step
  int64_t M = 0, K = 0;
  const fftc::ColEntry* ce = nullptr;
  const fftc::RowEntry* re = nullptr;
  float2* d_tw_row = nullptr;  // stage twiddles for K
  float2* d_twA = nullptr;     // w_N^t, t < 4096
  float2* d_twB = nullptr;     // w_N^{4096 h}
  float2* d_work = nullptr;    // N*batch complex
  // multi-pass TMA path (power-of-two N > 4096)
  fftc::PassPlanData pp;
  // L2-resident multi-pass path (power-of-two N in 2^13..2^21)
  fftc::L2PlanData l2;
  // runtime-schedule multi-pass path (7-smooth N > 4096 that is not a power of two)
  fftc::GPassPlanData gp;
  float2* gp_tables[3 * fftc::kMaxGPasses] = {};  // device tables owned by gp (const in GPassStage)
  // JIT-compiled single pass (prime factors > 7): kernel from the per-process cache
  const fftc::JitKernel* jk = nullptr;
  int jit_R[32] = {};
  int jit_S = 0;
  // direct DFT on tensor cores (opt-in): G_hi | G_lo image
  float* d_direct = nullptr;
  // host-buffer execution
  fftc::HostStage* hs = nullptr;
  // distributed six-step
  fftc::DistState* dist = nullptr;
};

namespace fftc {
// enqueue one transform set of `batch` transforms with explicit workspace (api.cu)
cudaError_t exec_local(const fftc_plan* p, const float2* in, float2* out, long long batch, float2* work,
                       cudaStream_t st);
// twiddle tables, host double -> device fp32 (api.cu)
float2* upload_stage_table(int64_t N, const int* R, int S, cudaError_t* err);
float2* upload_root_table(int64_t N, int64_t count, int64_t step, cudaError_t* err);
}  // namespace fftc
