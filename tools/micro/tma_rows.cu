// Microbenchmark: TMA tensor-load streaming rate versus the row width of the box (sm_100a).
// A 2 GiB input viewed as [16][4096 rows][4096 columns] of 8-byte elements (a 2^24-point pass's
// strided rows: 32 KB row pitch).  A persistent CTA per SM streams tiles of C adjacent columns x
// ROWS rows (ROWS * C * 8 bytes per tile, boxes of <= 256 rows) into NBUF shared buffers, refilling a
// buffer as soon as its tile has landed (no compute): the load rate the pass kernels' TMA
// front end can reach for 16/32/64/128-byte rows with one or more tiles in flight.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rows tma_rows.cu -lcuda && ./tma_rows
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_stream(const __grid_constant__ CUtensorMap tm, int C, int ROWS, int NBUF, long long tiles,
                         int tiles_per_rowblock, int rowblocks, int* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[4];
  const uint32_t bytes = (uint32_t)ROWS * C * 8u;
  if (threadIdx.x == 0)
    for (int k = 0; k < NBUF; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[k])));
  __syncthreads();
  auto issue = [&](long long t, int k) {
    // tile t: column group (t % tiles_per_rowblock), row block (t / tpr) % rowblocks, batch
    const int cg = (int)(t % tiles_per_rowblock);
    const long long rest = t / tiles_per_rowblock;
    const int rb = (int)(rest % rowblocks), b = (int)(rest / rowblocks);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[k])), "r"(bytes));
    for (int h = 0; h < ROWS; h += 256) {
      unsigned char* dst = sm + (size_t)k * bytes + (size_t)h * C * 8;
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              smem_u32(dst)),
          "l"(&tm), "r"(cg * C), "r"(rb * ROWS + h), "r"(b), "r"(smem_u32(&full[k]))
          : "memory");
    }
  };
  long long it = 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < NBUF; ++k)
      if (blockIdx.x + (long long)k * gridDim.x < tiles) issue(blockIdx.x + (long long)k * gridDim.x, k);
  int acc = 0;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
    const int k = (int)(it % NBUF);
    const uint32_t par = (uint32_t)((it / NBUF) & 1);
    asm volatile(
        "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&full[k])),
        "r"(par)
        : "memory");
    acc += sm[(size_t)k * bytes + threadIdx.x];
    __syncthreads();
    const long long tn = t + (long long)NBUF * gridDim.x;
    if (threadIdx.x == 0 && tn < tiles) issue(tn, k);
  }
  if (acc == 123456789) sink[0] = acc;
}

typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long long NB = 4096, L = 4096, B = 16;
  void* d = nullptr;
  int* sink = nullptr;
  cudaMalloc(&d, (size_t)NB * L * B * 8);
  cudaMalloc(&sink, 4);
  cudaMemset(d, 1, (size_t)NB * L * B * 8);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  encode_fn enc = (encode_fn)p;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int cfg[][3] = {  // C, ROWS, NBUF
      {2, 4096, 1}, {4, 4096, 1}, {8, 2048, 1}, {16, 1024, 1}, {4, 2048, 2}, {8, 1024, 2}, {16, 512, 2},
      {4, 1024, 3}, {8, 512, 3},  {16, 256, 3}, {4, 4096, 1}, {2, 4096, 1}};
  for (auto& c : cfg) {
    const int C = c[0], ROWS = c[1], NBUF = c[2];
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)NB, (cuuint64_t)L, (cuuint64_t)B};
    cuuint64_t strides[2] = {(cuuint64_t)NB * 8, (cuuint64_t)NB * L * 8};
    cuuint32_t box[3] = {(cuuint32_t)C, (cuuint32_t)(ROWS < 256 ? ROWS : 256), 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed C=%d\n", C);
      continue;
    }
    const size_t smem = (size_t)NBUF * ROWS * C * 8;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int tpr = (int)(NB / C), rbs = (int)(L / ROWS);
    const long long tiles = (long long)tpr * rbs * B;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      k_stream<<<sms, 128, smem>>>(tm, C, ROWS, NBUF, tiles, tpr, rbs, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    const cudaError_t err = cudaGetLastError();
    printf("{\"C\": %d, \"row_bytes\": %d, \"rows\": %d, \"nbuf\": %d, \"tile_kb\": %zu, \"ms\": %.4f, \"read_GBs\": %.1f, \"err\": \"%s\"}\n",
           C, C * 8, ROWS, NBUF, (size_t)ROWS * C * 8 / 1024, best, (double)NB * L * B * 8 / (best * 1e-3) / 1e9,
           cudaGetErrorString(err));
  }
  return 0;
}
