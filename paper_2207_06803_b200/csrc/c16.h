// c16.h -- N = 65536 in one HBM round trip on a cluster of eight CTAs (c16.cu), host side (product path).
#pragma once
#include <cuda_runtime.h>

namespace fftc {

bool c16_available();
// tw256: the DFT_256 stage table of radices [16, 16] (upload_stage_table(256, {16, 16}));
// twA: w_65536^t, t < 256; twB: w_65536^{256 h}, h <= 256
cudaError_t c16_execute(const float2* in, float2* out, long long batch, int conj, const float2* tw256,
                        const float2* twA, const float2* twB, cudaStream_t st);

}  // namespace fftc
