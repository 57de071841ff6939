// passes.h -- multi-pass (TMA tensor tile) large-N path, host side (product path).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fftc {

struct PassGeom {
  long long tiles_total;  // batch * tiles_per_batch
  int tiles_per_batch;    // (N / L) / cols
  int Ns;                 // Stockham Ns of this pass (product of earlier pass lengths)
  long long N;
  int tw;                 // apply the input twiddle w_{Ns L}^{(c mod Ns) r}
  int tws;                // twiddle table split: twA holds 2^tws entries
  int group;              // a CTA walks groups of this many adjacent tiles (1 = plain grid stride)
};

typedef cudaError_t (*pass_launch_fn)(bool first, const CUtensorMap& tin, const CUtensorMap& tout, float2* out_first,
                                      const float2* tw, const float2* twA, const float2* twB, const PassGeom& g,
                                      int conj_in, int conj_out, cudaStream_t st);

struct PassEntry {
  int L;
  int S;
  int R[8];
  int tpf;
  int cols;  // columns per tile (16: 128-byte rows; 8: 64-byte rows)
  pass_launch_fn launch;
  const char* name;
  int cluster = 0;  // > 0: a cluster of this many CTAs shares each tile's columns (cpass.cu)
};

// 4096-long pass on a cluster of four CTAs (cpass.cu): each CTA loads the rows = q (mod 4) of
// 8 columns through a 4-D tensor map (tin), writes its outputs straight to `out`
cudaError_t launch_cpass4096(bool first, const CUtensorMap& tin, const CUtensorMap& tout, float2* out,
                             const float2* tw, const float2* twA, const float2* twB, const PassGeom& g, int conj_in,
                             int conj_out, cudaStream_t st);

// 4096-long pass with the tile being computed held in registers (rpass.cu): 4-column tiles, the
// next tile's TMA load and a half-tile exchange buffer in shared memory, outputs stored by the threads
cudaError_t launch_rpass4096(bool first, const CUtensorMap& tin, const CUtensorMap& tout, float2* out,
                             const float2* tw, const float2* twA, const float2* twB, const PassGeom& g, int conj_in,
                             int conj_out, cudaStream_t st);
constexpr int kMaxPasses = 6;
struct PassPlanData {
  long long N = 0;
  int p = 0;
  const PassEntry* e[kMaxPasses] = {};
  float2* tw[kMaxPasses] = {};   // stage twiddles of DFT_{L_s}
  float2* twA[kMaxPasses] = {};  // w_{Ns L}^t, t < 2^tws
  float2* twB[kMaxPasses] = {};  // w_{Ns L}^{2^tws h}
  int tws[kMaxPasses] = {};      // split of the pass twiddle tables (balanced: ceil(log2(Ns L) / 2))
  int group[kMaxPasses] = {};    // tiles per CTA group (pass_group)
};

// Compiled pass kernel for length L (default per L, or a measured choice for the plan's N and
// the pass position -- first: the pass with Ns = 1; FFTC_PASS=<name>[,<name>...] overrides every
// pass of a listed length, FFTC_PASS_FIRST=<names> the first pass only).
const PassEntry* find_pass(int L, long long N = 0, bool first = false);
bool passes_available();
int pass_split(long long N, int* Ls, int max);
int pass_group(int L, long long N);
cudaError_t passes_execute(const PassPlanData& pp, const float2* in, float2* out, float2* work, long long batch,
                           int conj, cudaStream_t st);

}  // namespace fftc
