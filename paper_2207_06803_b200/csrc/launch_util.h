// launch_util.h -- one-time per-kernel launch setup (product path, host side).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace fftc {

// Dynamic shared-memory limit (and optionally the carveout) of a kernel plus its resident CTAs
// per SM, computed once.  Callers keep the result in a function-local `static const`, so the
// first call is thread-safe (C++11 static initialisation).  One process per GPU: the attributes
// are set on the device current at the first call.
struct KernelSetup {
  cudaError_t err;
  int grid_max;  // SMs x resident CTAs per SM (persistent grids)
};

template <class K>
KernelSetup kernel_setup(K kern, int threads, size_t smem, int carveout = -1, int per_sm = 0) {
  KernelSetup r{cudaSuccess, 0};
  r.err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (r.err == cudaSuccess && carveout >= 0)
    r.err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  if (r.err != cudaSuccess) return r;
  int dev = 0, sms = 0, per = per_sm;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (per <= 0) r.err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem);
  r.grid_max = sms * (per > 0 ? per : 1);
  return r;
}

}  // namespace fftc
