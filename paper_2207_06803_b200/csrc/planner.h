// planner.h -- radix planner (host only, product path).
#pragma once
#include <stdint.h>

namespace fftc {
bool seven_smooth(int64_t n);
// Generic schedule (codelet set of generic.cu); -1 if N is not 7-smooth.
int generic_radices(int64_t N, int* R, int max);
// Schedule used by the single-pass path: the compiled fast one if present, else generic.
int single_pass_radices(int64_t N, int* R, int max);
// 1: single pass (M = N, K = 1); 2: four-step N = M K; -1: unsupported.
int top_split(int64_t N, int64_t* M, int64_t* K);
}  // namespace fftc
