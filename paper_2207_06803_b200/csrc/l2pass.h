// l2pass.h -- L2-resident multi-pass path for large power-of-two N, host side (product path).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace fftc {

constexpr int kMaxL2Passes = 3;

struct L2Stage {  // one pass of the plan
  int L;          // pass length
  int which;      // 0: the kernel's long schedule, 1: its short one
  int Ns;         // product of the earlier pass lengths
  int T;          // column tiles (of 16) per transform = N / L / 16
  const float2* tw;   // stage twiddles of DFT_L
  const float2* twA;  // w_{Ns L}^t, t < 2^tws
  const float2* twB;  // w_{Ns L}^{2^tws h}
  int tws;            // twiddle table split
};

// Kernel parameters (one __grid_constant__ struct; the tensor maps must stay 64-byte aligned).
struct __align__(64) L2Params {
  CUtensorMap ld[kMaxL2Passes];  // ld[0]: input [B][L0][N/L0]; ld[s>0]: ring [slots*tc][Ls][N/Ls]
  CUtensorMap st[kMaxL2Passes];  // st[s>0]: autosort store, ring (s < p-1) or out (s = p-1)
  L2Stage ps[kMaxL2Passes];
  float2* ring;    // slots * tc * N complex (the pass intermediates; stays in L2)
  unsigned* ctr;   // [0] ticket; [1 + c p + s] tiles written; [1 + (nchunks + c) p + s] tiles read
  long long N, B;
  int p, tc, nchunks, slots, lag;
  float csign;     // -1: inverse (conjugate the input of pass 0 and the output of pass p-1)
};

typedef cudaError_t (*l2_launch_fn)(const L2Params& prm, cudaStream_t st);

struct L2Entry {
  int LA, LB;  // the two pass lengths one kernel instance handles (LA >= LB)
  l2_launch_fn launch;
  const char* name;
};

struct L2PlanData {
  long long N = 0;
  int p = 0;
  int L[kMaxL2Passes] = {};
  const L2Entry* e = nullptr;
  int tc = 0;       // transforms per chunk
  int slots = 0;    // ring slots of tc transforms
  int lag = 0;      // phases between consecutive passes of a chunk
  float2* tw[kMaxL2Passes] = {};
  float2* twA[kMaxL2Passes] = {};
  float2* twB[kMaxL2Passes] = {};
  int tws[kMaxL2Passes] = {};
};

// Pass lengths of the L2 path: p = 2 for 2^13..2^16, p = 3 for 2^17..2^21, each in
// {32, 64, 128, 256}, as equal as possible, longer first.  Returns p or -1.
int l2_split(long long N, int* Ls, int max);
// Kernel instance for the lengths, or NULL.
const L2Entry* find_l2(const int* Ls, int p);
// Transforms per chunk, ring slots and pass lag for N (env FFTC_L2_CHUNK_MB overrides the
// 8 MiB chunk, FFTC_L2_LAG the lag of 2 phases).
void l2_geometry(long long N, long long batch, int p, int* tc, int* slots, int* lag);
// Device bytes of the workspace (ring + counters) for `batch` transforms.
size_t l2_work_bytes(const L2PlanData& d, long long batch);
cudaError_t l2_execute(const L2PlanData& d, const float2* in, float2* out, void* work, long long batch, int conj,
                       cudaStream_t st);

}  // namespace fftc
