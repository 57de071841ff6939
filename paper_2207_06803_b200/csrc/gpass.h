// gpass.h -- runtime-schedule multi-pass path (any 7-smooth N > 4096), host side (product path).
#pragma once
#include <cuda_runtime.h>

#include "jit.h"
#include "registry.h"

namespace fftc {

constexpr int kGpassMaxL = 256;  // longest pass (16 columns x 257 x 2 buffers = 66 KB shared)
constexpr int kMaxGPasses = 4;

struct GPassStage {       // one pass (kernel argument)
  int L, Ns;              // pass length; product of the earlier pass lengths
  int S;                  // sub-stages of DFT_L
  int R[kMaxStages];      // their radices (generic codelet set)
  const float2* tw;       // stage twiddles of DFT_L
  const float2* twA;      // w_{Ns L}^t, t < 2^tws
  const float2* twB;      // w_{Ns L}^{2^tws h}
  int tws;                // balanced table split (both tables L1-resident)
  const JitKernel* jk;    // NVRTC kernel specialised to (L, radices), or null: k_gpass
};

struct GPassPlanData {
  long long N = 0;
  int p = 0;
  GPassStage st[kMaxGPasses] = {};
};

// Pass lengths for an N > 4096 whose prime factors are <= max_prime (7: compiled codelets;
// up to kJitMaxPrime with JIT pass kernels): the fewest passes (2..max) with every length
// <= kGpassMaxL, longest first.  Returns p or -1.
int gpass_split(long long N, int* Ls, int max, int max_prime = 7, int max_len = kGpassMaxL);
cudaError_t gpass_execute(const GPassPlanData& d, const float2* in, float2* out, float2* work, long long batch,
                          int conj, cudaStream_t st);

}  // namespace fftc
