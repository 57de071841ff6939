// registry.h -- table of compiled fused schedules (product path, host side).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fftc {

typedef cudaError_t (*batch_launch_fn)(const float2* in, float2* out, const float2* tw, long long batch,
                                       int conj, cudaStream_t st);

// One compiled single-pass schedule (fused.cuh, k_fused_batch).
struct FusedEntry {
  int N;
  int S;
  int R[8];
  int tpf, fpb, threads;
  int direct;  // 1: HBM I/O in the first/last stage (2: TMA bulk-copy fed, persistent; 3: register-pipelined, persistent); 0: staged through shared memory
  size_t smem;
  batch_launch_fn launch;
  const char* name;
};

// Fast schedules compiled for specific N (kernels_batch*.cu).  NULL if none.
const FusedEntry* find_fused(int N);
int fused_count();
const FusedEntry* fused_at(int i);

// Generic runtime-schedule kernel (generic.cu): any N <= kGenericMaxN whose
// radices are in the generic set.
constexpr int kGenericMaxN = 4096;
constexpr int kMaxStages = 16;
struct GenericSched {
  int N;
  int S;
  int R[kMaxStages];
};
cudaError_t launch_generic(const GenericSched& g, const float2* in, float2* out, const float2* tw,
                           long long batch, int conj, cudaStream_t st);
bool generic_supports_radix(int R);

}  // namespace fftc
