// dist.cu -- distributed six-step (placeholder until the NCCL path lands).
#include <stdio.h>

#include "dist.h"
#include "plan.h"

namespace fftc {
struct DistState {
  int dummy;
};
fftc_status dist_execute(DistState*, const void*, void*, cudaStream_t) { return FFTC_ERROR_UNSUPPORTED_SIZE; }
void dist_destroy(DistState* d) { delete d; }
int dist_launches(const DistState*) { return 0; }
int dist_describe(const DistState*, char* buf, size_t len) { return snprintf(buf, len, "kind=dist"); }
}  // namespace fftc

extern "C" fftc_status fftc_dist_get_unique_id(void*) { return FFTC_ERROR_NCCL; }
extern "C" fftc_plan* fftc_dist_plan_create(int64_t, int, const void*, int, int, int) { return nullptr; }
