// Microbenchmark: FP32 throughput of scalar FADD/FFMA vs packed FADD2/FFMA2 (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f32x2 f32x2.cu && ./f32x2
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

template <int MODE>
__global__ void k(float* out, int iters, float s) {
  float2 v[8];
  for (int i = 0; i < 8; ++i) v[i] = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
  const float2 w = make_float2(s, -s);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // scalar adds
        v[i].x = v[i].x + w.x; v[i].y = v[i].y + w.y;
      } else if (MODE == 1) {  // packed add
        u64 a = *reinterpret_cast<u64*>(&v[i]), b = *reinterpret_cast<const u64*>(&w);
        u64 r = add2(a, b);
        v[i] = *reinterpret_cast<float2*>(&r);
      } else if (MODE == 2) {  // scalar fma
        v[i].x = fmaf(v[i].x, w.x, w.y); v[i].y = fmaf(v[i].y, w.x, w.y);
      } else {  // packed fma
        u64 a = *reinterpret_cast<u64*>(&v[i]), b = *reinterpret_cast<const u64*>(&w);
        u64 r = fma2(a, b, b);
        v[i] = *reinterpret_cast<float2*>(&r);
      }
    }
  }
  float acc = 0;
  for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y;
  if (acc == 12345.f) out[0] = acc;
}

template <int MODE>
void run(const char* name) {
  float* out; cudaMalloc(&out, 4);
  const int iters = 1 << 14, blocks = 148 * 8, threads = 256;
  k<MODE><<<blocks, threads>>>(out, 16, 1e-7f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<blocks, threads>>>(out, iters, 1e-7f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double lane_ops = (double)blocks * threads * iters * 16;  // fp32 lane operations
  printf("{\"mode\": \"%s\", \"ms\": %.3f, \"G_fp32_lane_ops_per_s\": %.1f}\n", name, ms, lane_ops / ms / 1e6);
  cudaFree(out);
}

int main() {
  run<0>("fadd");
  run<1>("fadd2");
  run<2>("ffma");
  run<3>("ffma2");
  return 0;
}
