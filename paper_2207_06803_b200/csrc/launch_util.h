// launch_util.h -- one-time per-kernel launch setup (product path, host side).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include <mutex>

namespace fftc {

// Dynamic shared-memory limit (and optionally the carveout) of a kernel plus its resident CTAs
// per SM, computed once per device (callers keep it in a function-local PerDevice).
struct KernelSetup {
  cudaError_t err;
  int grid_max;  // SMs x resident CTAs per SM (persistent grids)
};

// One value per device, computed on first use on that device (thread-safe).  Kernel attributes
// (the dynamic shared-memory opt-in) are per device: a process that drives several GPUs must set
// them on each, so launchers keep their one-time setup in a function-local PerDevice.
constexpr int kMaxDevices = 64;

template <class T>
struct PerDevice {
  T v[kMaxDevices];
  std::once_flag once[kMaxDevices];
  template <class F>
  const T& get(F make) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    std::call_once(once[dev], [&] { v[dev] = make(); });
    return v[dev];
  }
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
