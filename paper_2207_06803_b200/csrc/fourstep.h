// fourstep.h -- compiled large-N pass kernels (product path, host side).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "colgeom.h"

namespace fftc {

typedef cudaError_t (*colx_launch_fn)(const float2* in, float2* out, const float2* tw, const float2* twA,
                                      const float2* twB, const ColGeom& g, long long groups, int conj_in,
                                      int conj_out, cudaStream_t st);
typedef cudaError_t (*row_launch_fn)(const float2* work, float2* out, const float2* tw, int M, long long N,
                                     long long batch, int conj, cudaStream_t st);

// DFT_M down C adjacent columns per CTA (colfft.cuh).  launch: lanes-walk-columns
// output; launch_t: transposed (shared-memory staged) output, or NULL.
struct ColEntry {
  int M;
  int S;
  int R[8];
  int tpf, cols;
  size_t smem, smem_t;
  colx_launch_fn launch;
  colx_launch_fn launch_t;
  const char* name;
};
// DFT_K along FPB rows per CTA + transposed store X[j + M k1] (four-step pass 2).
struct RowEntry {
  int K;
  int S;
  int R[8];
  int tpf, rows;
  size_t smem;
  row_launch_fn launch;
  const char* name;
};

const ColEntry* find_col(int M);
const RowEntry* find_row(int K);
int col_count();
int row_count();
const ColEntry* col_at(int i);
const RowEntry* row_at(int i);

// four-step pass-1 geometry for N = M K, batch transforms: columns r < K, stride K
ColGeom fourstep_cols_geom(const ColEntry* c, long long N, long long K);

}  // namespace fftc
