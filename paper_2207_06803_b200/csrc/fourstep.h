// fourstep.h -- compiled four-step pass kernels (product path, host side).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fftc {

typedef cudaError_t (*col_launch_fn)(const float2* in, float2* work, const float2* tw, const float2* twA,
                                     const float2* twB, int K, long long N, long long batch, int conj,
                                     cudaStream_t st);
typedef cudaError_t (*row_launch_fn)(const float2* work, float2* out, const float2* tw, int M, long long N,
                                     long long batch, int conj, cudaStream_t st);

// Pass 1: DFT_M down C adjacent columns per CTA (+ D^N_M twiddle).
struct ColEntry {
  int M;
  int S;
  int R[8];
  int tpf, cols;
  size_t smem;
  col_launch_fn launch;
};
// Pass 2: DFT_K along FPB rows per CTA + transposed store.
struct RowEntry {
  int K;
  int S;
  int R[8];
  int tpf, rows;
  size_t smem;
  row_launch_fn launch;
};

const ColEntry* find_col(int M);
const RowEntry* find_row(int K);
int col_count();
int row_count();
const ColEntry* col_at(int i);
const RowEntry* row_at(int i);

}  // namespace fftc
