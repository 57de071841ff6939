// dist.h -- distributed six-step plan state (product path, host side).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "../../include/fftc.h"

namespace fftc {
struct DistState;
fftc_status dist_execute(DistState* d, const void* in, void* out, cudaStream_t st);
void dist_destroy(DistState* d);
int dist_launches(const DistState* d);
int dist_describe(const DistState* d, char* buf, size_t len);
}  // namespace fftc
