// direct_tc.h -- direct DFT (dense product) on tcgen05 tensor cores, host side (product path).
#pragma once
#include <cuda_runtime.h>

namespace fftc {

// Sizes the tensor-core direct DFT is compiled for.
bool direct_supported(long long N);
// G_hi / G_lo (3xTF32 split of the real 2N x 2N DFT matrix for `sign`) in the swizzled
// shared-memory image the kernel bulk-copies; device allocation owned by the plan.
float* direct_tables(long long N, int sign, cudaError_t* err);
cudaError_t direct_execute(long long N, const float2* in, float2* out, const float* g_img, long long batch,
                           cudaStream_t st);

}  // namespace fftc
