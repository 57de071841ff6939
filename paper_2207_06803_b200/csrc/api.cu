// api.cu -- the C ABI of libfftc.so (include/fftc.h) (product path).
//
// Plan creation = planner (planner.cpp) + fp32 twiddle tables computed in double
// on the host + workspace; execution = stream-ordered kernel launches only.
// The inverse transform (sign = +1) runs the forward kernels on conjugated
// input and conjugates the output (IDFT x = conj(DFT(conj x))), so every table
// and codelet is the forward w_N = exp(-2 pi i / N) of PAPER.md P:46.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/fftc.h"
#include "dist.h"
#include "expr.h"
#include "plan.h"
#include "planner.h"

using namespace fftc;

static thread_local fftc_status g_last = FFTC_SUCCESS;

namespace fftc {

static void root(int64_t e, int64_t L, float2* out) {
  // w_L^e (forward), exponent reduced mod L in integers, angle taken in double
  e %= L;
  if (e < 0) e += L;
  const double a = 2.0 * M_PI * (double)e / (double)L;
  out->x = (float)cos(a);
  out->y = (float)(-sin(a));
}

float2* upload_stage_table(int64_t N, const int* R, int S, cudaError_t* err) {
  std::vector<float2> t((size_t)(N > 1 ? N : 1), make_float2(1.f, 0.f));
  int64_t Ns = 1;
  for (int s = 0; s < S; ++s) {
    const int64_t L = Ns * R[s];
    if (s > 0)
      for (int r = 1; r < R[s]; ++r)
        for (int64_t m = 0; m < Ns; ++m) root(m * r, L, &t[(size_t)((Ns - 1) + (r - 1) * Ns + m)]);
    Ns = L;
  }
  float2* d = nullptr;
  *err = cudaMalloc(&d, t.size() * sizeof(float2));
  if (*err != cudaSuccess) return nullptr;
  *err = cudaMemcpy(d, t.data(), t.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (*err != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  return d;
}

// entries w_N^{h * step} for h < count
float2* upload_root_table(int64_t N, int64_t count, int64_t step, cudaError_t* err) {
  std::vector<float2> t((size_t)count);
  for (int64_t h = 0; h < count; ++h) root(h * step, N, &t[(size_t)h]);
  float2* d = nullptr;
  *err = cudaMalloc(&d, t.size() * sizeof(float2));
  if (*err != cudaSuccess) return nullptr;
  *err = cudaMemcpy(d, t.data(), t.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (*err != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  return d;
}

// split of a two-level root table for w_T^e, e < T: 2^sh low entries, T / 2^sh + 1 high ones
int balanced_split(int64_t T) {
  int n = 0;
  while (((int64_t)1 << n) < T) ++n;
  return (n + 1) / 2;
}

cudaError_t exec_local(const fftc_plan* p, const float2* in, float2* out, long long batch, float2* work,
                       cudaStream_t st) {
  const int conj = p->sign > 0;
  switch (p->kind) {
    case KIND_COPY:
      return cudaMemcpyAsync(out, in, (size_t)batch * p->N * sizeof(float2), cudaMemcpyDeviceToDevice, st);
    case KIND_FUSED:
      return p->fe->launch(in, out, p->d_tw, batch, conj, st);
    case KIND_GENERIC:
      return launch_generic(p->gs, in, out, p->d_tw, batch, conj, st);
    case KIND_PASSES:
      return passes_execute(p->pp, in, out, work, batch, conj, st);
    case KIND_L2:
      return l2_execute(p->l2, in, out, work, batch, conj, st);
    case KIND_GPASS:
      return gpass_execute(p->gp, in, out, work, batch, conj, st);
    case KIND_JIT:
      return jit_launch(p->jk, in, out, p->d_tw, batch, conj, st);
    case KIND_DIRECT:
      return direct_execute(p->N, in, out, p->d_direct, batch, st);
    case KIND_CLUSTER:
      return c16_execute(in, out, batch, conj, p->d_tw, p->d_twA, p->d_twB, st);

    case KIND_FOURSTEP: {
      const ColGeom g = fourstep_cols_geom(p->ce, p->N, p->K);
      cudaError_t e = p->ce->launch(in, work, p->d_tw, p->d_twA, p->d_twB, g, batch, conj, 0, st);
      if (e != cudaSuccess) return e;
      return p->re->launch(work, out, p->d_tw_row, (int)p->M, p->N, batch, conj, st);
    }
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace fftc

static fftc_status from_cuda(cudaError_t e) {
  if (e == cudaSuccess) return FFTC_SUCCESS;
  if (e == cudaErrorMemoryAllocation) return FFTC_ERROR_OUT_OF_MEMORY;
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return FFTC_ERROR_NO_DEVICE;
  return FFTC_ERROR_CUDA;
}

static void free_host_stage(fftc::HostStage* hs) {
  if (!hs) return;
  for (int i = 0; i < HostStage::kDepth; ++i) {
    cudaFree(hs->d_in[i]);
    cudaFree(hs->d_out[i]);
    cudaFree(hs->d_work[i]);
    if (hs->st[i]) cudaStreamDestroy(hs->st[i]);
  }
  delete hs;
}

static void free_plan(fftc_plan* p) {
  if (!p) return;
  if (p->dist) dist_destroy(p->dist);
  cudaFree(p->d_tw);
  cudaFree(p->d_tw_row);
  cudaFree(p->d_twA);
  cudaFree(p->d_twB);
  cudaFree(p->d_work);
  for (int i = 0; i < 3 * kMaxGPasses; ++i) cudaFree(p->gp_tables[i]);
  cudaFree(p->d_direct);
  for (int s = 0; s < kMaxL2Passes; ++s) {
    cudaFree(p->l2.tw[s]);
    cudaFree(p->l2.twA[s]);
    cudaFree(p->l2.twB[s]);
  }
  for (int s = 0; s < kMaxPasses; ++s) {
    cudaFree(p->pp.tw[s]);
    cudaFree(p->pp.twA[s]);
    cudaFree(p->pp.twB[s]);
  }
  free_host_stage(p->hs);
  delete p;
}

static void free_plan(fftc_plan* p);

// Runtime-schedule passes (gpass.cu) with explicit lengths and per-pass radices.  Each pass
// gets an NVRTC kernel specialised to (L, radices) when NVRTC is there (FFTC_GPASS_JIT=0
// keeps the compiled runtime-schedule kernel); radices outside the compiled codelet set need it.
static fftc_status setup_gpass(fftc_plan* p, const int* Lg, int pg, const int (*R)[kMaxStages], const int* S) {
  cudaError_t err = cudaSuccess;
  const char* ej = getenv("FFTC_GPASS_JIT");
  const bool try_jit = jit_available() && !(ej && strcmp(ej, "0") == 0);
  p->kind = KIND_GPASS;
  p->gp.N = p->N;
  p->gp.p = pg;
  int64_t Ns = 1;
  for (int s = 0; s < pg && err == cudaSuccess; ++s) {
    GPassStage& g = p->gp.st[s];
    g.L = Lg[s];
    g.Ns = (int)Ns;
    g.S = S[s];
    g.jk = nullptr;
    if (g.L > kJitPassMaxL || g.S < 1 || g.S > kMaxStages) return FFTC_ERROR_UNSUPPORTED_SIZE;
    int64_t prod = 1;
    bool generic = true;
    for (int t = 0; t < g.S; ++t) {
      generic = generic && generic_supports_radix(R[s][t]);
      g.R[t] = R[s][t];
      prod *= R[s][t];
    }
    if (prod != g.L) return FFTC_ERROR_INVALID_VALUE;
    if (try_jit) {
      cudaError_t je = cudaSuccess;
      g.jk = jit_pass_get(g.L, g.R, g.S, &je);
    }
    if (!g.jk && (!generic || g.L > kGpassMaxL)) return FFTC_ERROR_UNSUPPORTED_SIZE;
    const int64_t T = Ns * Lg[s];
    float2* t0 = upload_stage_table(Lg[s], g.R, g.S, &err);
    p->gp_tables[3 * s] = t0;
    g.tw = t0;
    g.tws = balanced_split(T);
    if (err == cudaSuccess) {
      float2* t1 = upload_root_table(T, (int64_t)1 << g.tws, 1, &err);
      p->gp_tables[3 * s + 1] = t1;
      g.twA = t1;
    }
    if (err == cudaSuccess) {
      float2* t2 = upload_root_table(T, (T >> g.tws) + 1, (int64_t)1 << g.tws, &err);
      p->gp_tables[3 * s + 2] = t2;
      g.twB = t2;
    }
    Ns = T;
  }
  if (err == cudaSuccess && p->batch > 0 && pg > 1)
    err = cudaMalloc(&p->d_work, (size_t)(p->N * p->batch) * sizeof(float2));
  return from_cuda(err);
}

static fftc_plan* fail(fftc_plan* p, fftc_status s) {
  free_plan(p);
  g_last = s;
  return nullptr;
}

extern "C" void fftc_set_last_error(fftc_status s) { g_last = s; }

extern "C" fftc_status fftc_check_device(int* dev) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return FFTC_ERROR_NO_DEVICE;
  if (cudaGetDevice(dev) != cudaSuccess) return FFTC_ERROR_NO_DEVICE;
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, *dev);
  if (major != 10) return FFTC_ERROR_NO_DEVICE;  // kernels are sm_100a only
  return FFTC_SUCCESS;
}

extern "C" {

fftc_plan* fftc_plan_create(int64_t N, int64_t batch, int sign) {
  g_last = FFTC_SUCCESS;
  if (N < 1 || batch < 0 || (sign != -1 && sign != 1)) return fail(nullptr, FFTC_ERROR_INVALID_VALUE);
  int Rj[32];
  const int Sj = seven_smooth(N) ? -1 : (N <= kGenericMaxN ? jit_radices((int)N, Rj, 32) : -1);
  int Lj[kMaxGPasses];
  const int pj = (!seven_smooth(N) && N > kGenericMaxN)
                     ? gpass_split(N, Lj, kMaxGPasses, kJitMaxPrime, kGpassSplitMaxL)
                     : -1;
  if (!seven_smooth(N) && Sj < 0 && pj < 0) return fail(nullptr, FFTC_ERROR_UNSUPPORTED_SIZE);
  if (batch > 0 && batch > ((int64_t)1 << 60) / (N * 8)) return fail(nullptr, FFTC_ERROR_UNSUPPORTED_SIZE);
  int dev = 0;
  fftc_status ds = fftc_check_device(&dev);
  if (ds != FFTC_SUCCESS) return fail(nullptr, ds);
  fftc_plan* p = new fftc_plan();
  p->N = N;
  p->batch = batch;
  p->sign = sign;
  p->device = dev;
  cudaError_t err = cudaSuccess;
  if (pj > 0) {
    // above 4096 with prime factors 11..61: runtime passes, each an NVRTC-specialised kernel
    if (!jit_available()) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
    int R[kMaxGPasses][kMaxStages], S[kMaxGPasses];
    for (int s = 0; s < pj; ++s) {
      int tmp[32];
      S[s] = jit_pass_radices(Lj[s], tmp, 32);
      if (S[s] < 1 || S[s] > kMaxStages) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
      for (int t = 0; t < S[s]; ++t) R[s][t] = tmp[t];
    }
    const fftc_status st = setup_gpass(p, Lj, pj, R, S);
    return st == FFTC_SUCCESS ? p : fail(p, st);
  }
  if (Sj > 0) {
    // prime factors > 7: a kernel generated for N and compiled now (NVRTC, sm_100a)
    if (!jit_available()) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
    p->kind = KIND_JIT;
    p->jit_S = Sj;
    for (int s = 0; s < Sj; ++s) p->jit_R[s] = Rj[s];
    p->jk = jit_get((int)N, &err);
    if (!p->jk) return fail(p, err == cudaErrorNotSupported ? FFTC_ERROR_UNSUPPORTED_SIZE : from_cuda(err));
    p->d_tw = upload_stage_table(N, Rj, Sj, &err);
    if (err != cudaSuccess) return fail(p, from_cuda(err));
    return p;
  }
  if (N == 1) {
    p->kind = KIND_COPY;
    return p;
  }
  int64_t M = 0, K = 0;
  const int split = top_split(N, &M, &K);
  if (split == 1) {
    int R[kMaxStages];
    // FFTC_FORCE_JIT=1 (tuning): the generated kernel even where a compiled schedule exists
    const char* fj = getenv("FFTC_FORCE_JIT");
    const FusedEntry* fe = (fj && strcmp(fj, "1") == 0) ? nullptr : find_fused((int)N);
    // 7-smooth N without a compiled schedule: a kernel generated for N (NVRTC; measured 3.3-6.2x
    // faster than the compiled runtime-schedule kernel, profiles/r02c/smooth_jit.jsonl), unless
    // NVRTC is missing or FFTC_SMOOTH_JIT=0
    const char* sj = getenv("FFTC_SMOOTH_JIT");
    const bool smooth_jit = !fe && jit_available() && !(sj && strcmp(sj, "0") == 0);
    int Rs[32];
    const int Ss = smooth_jit ? jit_radices((int)N, Rs, 32) : -1;
    const JitKernel* jk = Ss > 0 ? jit_get((int)N, &err) : nullptr;
    err = cudaSuccess;  // a generated kernel that cannot be built falls back to the compiled one
    if (jk) {
      p->kind = KIND_JIT;
      p->jit_S = Ss;
      for (int s = 0; s < Ss; ++s) p->jit_R[s] = Rs[s];
      p->jk = jk;
      p->d_tw = upload_stage_table(N, Rs, Ss, &err);
    } else if (fe) {
      p->kind = KIND_FUSED;
      p->fe = fe;
      p->d_tw = upload_stage_table(N, fe->R, fe->S, &err);
    } else {
      const int S = generic_radices(N, R, kMaxStages);
      if (S < 0 || S > kMaxStages) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
      p->kind = KIND_GENERIC;
      p->gs.N = (int)N;
      p->gs.S = S;
      for (int s = 0; s < S; ++s) p->gs.R[s] = R[s];
      p->d_tw = upload_stage_table(N, R, S, &err);
    }
    if (err != cudaSuccess) return fail(p, from_cuda(err));
    return p;
  }
  const char* large = getenv("FFTC_LARGE");
  // L2-resident multi-pass path (FFTC_LARGE=l2): powers of two 2^13..2^21, one HBM round
  // trip.  Measured on B200 (profiles/r01d): the pass tiles are issue-bound (~60 thread
  // instructions per element per pass), so running all passes in one kernel does not beat
  // the HBM multi-pass kernels yet; it is opt-in until the tile compute is cheaper.
  {
    int Ls2[kMaxL2Passes];
    const int np2 = l2_split(N, Ls2, kMaxL2Passes);
    const L2Entry* e2 = np2 > 0 ? find_l2(Ls2, np2) : nullptr;
    const bool want = large && strcmp(large, "l2") == 0;
    if (e2 && want && passes_available()) {
      p->kind = KIND_L2;
      L2PlanData& d = p->l2;
      d.N = N;
      d.p = np2;
      d.e = e2;
      l2_geometry(N, batch, np2, &d.tc, &d.slots, &d.lag);
      int64_t Ns = 1;
      for (int s = 0; s < np2 && err == cudaSuccess; ++s) {
        d.L[s] = Ls2[s];
        const PassEntry* pe = find_pass(Ls2[s]);  // same radices as the HBM pass kernel of this length
        if (!pe) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
        const int64_t T = Ns * Ls2[s];
        d.tw[s] = upload_stage_table(Ls2[s], pe->R, pe->S, &err);
        d.tws[s] = balanced_split(T);
        if (err == cudaSuccess) d.twA[s] = upload_root_table(T, (int64_t)1 << d.tws[s], 1, &err);
        if (err == cudaSuccess)
          d.twB[s] = upload_root_table(T, (T >> d.tws[s]) + 1, (int64_t)1 << d.tws[s], &err);
        Ns = T;
      }
      if (err == cudaSuccess && batch > 0) err = cudaMalloc(&p->d_work, l2_work_bytes(d, batch));
      if (err != cudaSuccess) return fail(p, from_cuda(err));
      return p;
    }
  }
  // N = 65536 in one HBM round trip on a cluster of eight CTAs (c16.cu; FFTC_LARGE=cluster)
  if (N == 65536 && large && strcmp(large, "cluster") == 0 && c16_available()) {
    p->kind = KIND_CLUSTER;
    const int R16[2] = {16, 16};
    p->d_tw = upload_stage_table(256, R16, 2, &err);
    if (err == cudaSuccess) p->d_twA = upload_root_table(65536, 256, 1, &err);
    if (err == cudaSuccess) p->d_twB = upload_root_table(65536, 257, 256, &err);
    if (err != cudaSuccess) return fail(p, from_cuda(err));
    return p;
  }
  // multi-pass TMA path for powers of two (FFTC_LARGE=fourstep selects the two-pass kernels)
  int Ls[kMaxPasses];
  const int np = pass_split(N, Ls, kMaxPasses);
  // measured on B200 (profiles/r01d): with shared-state-space tile addressing the TMA passes
  // beat the four-step at every power of two above 4096 (2^20: three passes 2.37 ms vs the
  // 512 x 2048 four-step 2.55 ms per 2^28 elements)
  bool use_passes = np > 0 && passes_available();
  if (large && strcmp(large, "fourstep") == 0) use_passes = false;
  if (large && strcmp(large, "passes") == 0 && np > 0 && passes_available()) use_passes = true;
  if (large && strcmp(large, "gpass") == 0) use_passes = false;
  if (use_passes) {
    p->kind = KIND_PASSES;
    p->pp.N = N;
    p->pp.p = np;
    int64_t Ns = 1;
    for (int s = 0; s < np && err == cudaSuccess; ++s) {
      const PassEntry* e = find_pass(Ls[s], N, s == 0);
      if (!e) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
      p->pp.e[s] = e;
      const int64_t T = Ns * Ls[s];
      p->pp.tw[s] = upload_stage_table(Ls[s], e->R, e->S, &err);
      p->pp.tws[s] = balanced_split(T);
      p->pp.group[s] = pass_group(Ls[s], N);
      if (err == cudaSuccess) p->pp.twA[s] = upload_root_table(T, (int64_t)1 << p->pp.tws[s], 1, &err);
      if (err == cudaSuccess)
        p->pp.twB[s] = upload_root_table(T, (T >> p->pp.tws[s]) + 1, (int64_t)1 << p->pp.tws[s], &err);
      Ns = T;
    }
    if (err == cudaSuccess && batch > 0 && np > 1) err = cudaMalloc(&p->d_work, (size_t)(N * batch) * sizeof(float2));
    if (err != cudaSuccess) return fail(p, from_cuda(err));
    return p;
  }
  // any other 7-smooth N (and FFTC_LARGE=gpass): runtime-schedule multi-pass kernels
  const bool force_gpass = large && strcmp(large, "gpass") == 0;
  if (np < 0 || force_gpass) {
    const char* ej = getenv("FFTC_GPASS_JIT");
    const bool jit = jit_available() && !(ej && strcmp(ej, "0") == 0);
    int Lg[kMaxGPasses];
    // JIT passes run lengths up to kGpassSplitMaxL = 512 (fewer HBM passes); the compiled kernel 256
    const int pg = gpass_split(N, Lg, kMaxGPasses, 7, jit ? kGpassSplitMaxL : kGpassMaxL);
    if (pg < 0) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
    int R[kMaxGPasses][kMaxStages], S[kMaxGPasses];
    for (int s = 0; s < pg; ++s)  // JIT passes: balanced radices; compiled kernel: the generic set
      S[s] = jit ? jit_pass_radices(Lg[s], R[s], kMaxStages) : generic_radices(Lg[s], R[s], kMaxStages);
    const fftc_status st = setup_gpass(p, Lg, pg, R, S);
    return st == FFTC_SUCCESS ? p : fail(p, st);
  }
  // four-step
  if (split < 0) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
  p->kind = KIND_FOURSTEP;
  p->M = M;
  p->K = K;
  p->ce = find_col((int)M);
  p->re = find_row((int)K);
  if (!p->ce || !p->re) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
  p->d_tw = upload_stage_table(M, p->ce->R, p->ce->S, &err);
  if (err == cudaSuccess) p->d_tw_row = upload_stage_table(K, p->re->R, p->re->S, &err);
  const int64_t nA = N < 4096 ? N : 4096;
  if (err == cudaSuccess) p->d_twA = upload_root_table(N, nA, 1, &err);
  if (err == cudaSuccess) p->d_twB = upload_root_table(N, (N + 4095) / 4096, 4096, &err);
  if (err == cudaSuccess && batch > 0) err = cudaMalloc(&p->d_work, (size_t)(N * batch) * sizeof(float2));
  if (err != cudaSuccess) return fail(p, from_cuda(err));
  return p;
}

static bool misaligned(const void* a) { return ((uintptr_t)a & 15u) != 0; }

// A plan's tables, workspace and kernel attributes live on the device current at create.
static bool on_plan_device(const fftc_plan* p) {
  int dev = -1;
  return cudaGetDevice(&dev) == cudaSuccess && dev == p->device;
}

fftc_status fftc_execute(const fftc_plan* p, const void* in, void* out, void* stream) {
  if (!p || !in || !out) return FFTC_ERROR_INVALID_VALUE;
  if (!on_plan_device(p)) return FFTC_ERROR_WRONG_DEVICE;
  if (p->kind == KIND_DIST) return dist_execute(p->dist, in, out, (cudaStream_t)stream);
  if (p->batch == 0) return FFTC_SUCCESS;
  const size_t bytes = (size_t)(p->N * p->batch) * sizeof(float2);
  const char* a = (const char*)in;
  const char* b = (const char*)out;
  if (a < b + bytes && b < a + bytes) return FFTC_ERROR_INVALID_VALUE;  // in-place / overlap
  if (misaligned(in) || misaligned(out)) return FFTC_ERROR_MISALIGNED;
  cudaError_t e = cudaGetLastError();  // report an earlier asynchronous fault
  if (e != cudaSuccess) return from_cuda(e);
  e = exec_local(p, (const float2*)in, (float2*)out, p->batch, p->d_work, (cudaStream_t)stream);
  return from_cuda(e);
}

fftc_status fftc_execute_host(fftc_plan* p, const void* host_in, void* host_out) {
  if (!p || !host_in || !host_out || host_in == host_out) return FFTC_ERROR_INVALID_VALUE;
  if (p->kind == KIND_DIST) return FFTC_ERROR_INVALID_VALUE;
  if (!on_plan_device(p)) return FFTC_ERROR_WRONG_DEVICE;
  if (p->batch == 0) return FFTC_SUCCESS;
  const int64_t tbytes = p->N * (int64_t)sizeof(float2);
  cudaError_t e = cudaSuccess;
  if (!p->hs) {
    HostStage* hs = new HostStage();
    p->hs = hs;
    // ~32 MiB per chunk, at least one transform
    int64_t chunk_bytes = (int64_t)32 << 20;  // tuning: FFTC_HOST_CHUNK_MB, FFTC_HOST_DEPTH
    if (const char* c = getenv("FFTC_HOST_CHUNK_MB")) chunk_bytes = atoll(c) << 20;
    if (const char* dpt = getenv("FFTC_HOST_DEPTH")) hs->depth = atoi(dpt);
    if (hs->depth < 2) hs->depth = 2;
    if (hs->depth > HostStage::kDepth) hs->depth = HostStage::kDepth;
    int64_t chunk = chunk_bytes / tbytes;
    if (chunk < 1) chunk = 1;
    if (chunk > p->batch) chunk = p->batch;
    hs->chunk = chunk;
    for (int i = 0; i < hs->depth && e == cudaSuccess; ++i) {
      e = cudaMalloc(&hs->d_in[i], (size_t)(chunk * tbytes));
      if (e == cudaSuccess) e = cudaMalloc(&hs->d_out[i], (size_t)(chunk * tbytes));
      if (e == cudaSuccess && (p->kind == KIND_FOURSTEP || p->kind == KIND_PASSES || p->kind == KIND_GPASS))
        e = cudaMalloc(&hs->d_work[i], (size_t)(chunk * tbytes));
      if (e == cudaSuccess && p->kind == KIND_L2) e = cudaMalloc(&hs->d_work[i], l2_work_bytes(p->l2, chunk));
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&hs->st[i], cudaStreamNonBlocking);
    }
    if (e != cudaSuccess) {  // leave no half-built staging area behind: the next call retries
      free_host_stage(hs);
      p->hs = nullptr;
      return from_cuda(e);
    }
  }
  HostStage* hs = p->hs;
  const char* hin = (const char*)host_in;
  char* hout = (char*)host_out;
  // chunk sizes ramp up from chunk/8 and back down at the end, so the first H2D and the last
  // D2H -- the two copies nothing overlaps -- are short (pipeline fill and drain)
  const int64_t cmin = hs->chunk / 8 > 0 ? hs->chunk / 8 : 1;
  int64_t ramp = cmin;
  int k = 0;
  int64_t nb = 0;
  for (int64_t t0 = 0; t0 < p->batch && e == cudaSuccess; t0 += nb, k = (k + 1) % hs->depth) {
    const int64_t rem = p->batch - t0;
    nb = ramp;
    if (ramp < hs->chunk) ramp = 2 * ramp < hs->chunk ? 2 * ramp : hs->chunk;  // ramp up, capped
    if (rem <= 2 * hs->chunk) nb = rem / 2 > cmin ? rem / 2 : cmin;  // ramp down: halves
    if (nb > rem) nb = rem;
    if (nb < 1 || nb > hs->chunk) {  // staging buffers hold hs->chunk transforms
      e = cudaErrorInvalidValue;
      break;
    }
    const size_t bytes = (size_t)(nb * tbytes);
    e = cudaMemcpyAsync(hs->d_in[k], hin + t0 * tbytes, bytes, cudaMemcpyHostToDevice, hs->st[k]);
    if (e == cudaSuccess) e = exec_local(p, hs->d_in[k], hs->d_out[k], nb, hs->d_work[k], hs->st[k]);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(hout + t0 * tbytes, hs->d_out[k], bytes, cudaMemcpyDeviceToHost, hs->st[k]);
  }
  for (int i = 0; i < hs->depth; ++i) {
    cudaError_t s = cudaStreamSynchronize(hs->st[i]);
    if (e == cudaSuccess) e = s;
  }
  return from_cuda(e);
}

void fftc_plan_destroy(fftc_plan* p) { free_plan(p); }

fftc_status fftc_last_error(void) { return g_last; }

const char* fftc_status_string(fftc_status s) {
  switch (s) {
    case FFTC_SUCCESS: return "FFTC_SUCCESS";
    case FFTC_ERROR_INVALID_VALUE: return "FFTC_ERROR_INVALID_VALUE";
    case FFTC_ERROR_UNSUPPORTED_SIZE: return "FFTC_ERROR_UNSUPPORTED_SIZE";
    case FFTC_ERROR_MISALIGNED: return "FFTC_ERROR_MISALIGNED";
    case FFTC_ERROR_OUT_OF_MEMORY: return "FFTC_ERROR_OUT_OF_MEMORY";
    case FFTC_ERROR_CUDA: return "FFTC_ERROR_CUDA";
    case FFTC_ERROR_NCCL: return "FFTC_ERROR_NCCL";
    case FFTC_ERROR_NO_DEVICE: return "FFTC_ERROR_NO_DEVICE";
    case FFTC_ERROR_WRONG_DEVICE: return "FFTC_ERROR_WRONG_DEVICE";
  }
  return "FFTC_UNKNOWN";
}

int fftc_plan_launches(const fftc_plan* p) {
  if (!p) return -1;
  switch (p->kind) {
    case KIND_COPY: return 0;
    case KIND_FUSED:
    case KIND_GENERIC: return p->batch > 0 ? 1 : 0;
    case KIND_FOURSTEP: return p->batch > 0 ? 2 : 0;
    case KIND_PASSES: return p->batch > 0 ? p->pp.p : 0;
    case KIND_L2: return p->batch > 0 ? 1 : 0;
    case KIND_GPASS: return p->batch > 0 ? p->gp.p : 0;
    case KIND_JIT: return p->batch > 0 ? 1 : 0;
    case KIND_DIRECT: return p->batch > 0 ? 1 : 0;
    case KIND_CLUSTER: return p->batch > 0 ? 1 : 0;
    case KIND_DIST: return dist_launches(p->dist);
  }
  return -1;
}

int fftc_plan_describe(const fftc_plan* p, char* buf, size_t len) {
  if (!p) return -1;
  char tmp[512];
  int n = 0;
  auto rad = [&](const int* R, int S) {
    for (int s = 0; s < S; ++s) n += snprintf(tmp + n, sizeof(tmp) - n, "%s%d", s ? "x" : "", R[s]);
  };
  switch (p->kind) {
    case KIND_COPY:
      n += snprintf(tmp + n, sizeof(tmp) - n, "kind=copy N=%lld batch=%lld", (long long)p->N, (long long)p->batch);
      break;
    case KIND_FUSED:
      n += snprintf(tmp + n, sizeof(tmp) - n, "kind=fused N=%lld batch=%lld sign=%d radices=", (long long)p->N,
                    (long long)p->batch, p->sign);
      rad(p->fe->R, p->fe->S);
      n += snprintf(tmp + n, sizeof(tmp) - n, " kernel=%s tpf=%d fpb=%d io=%s smem=%zu launches=1", p->fe->name,
                    p->fe->tpf, p->fe->fpb, p->fe->direct ? "direct" : "staged", p->fe->smem);
      break;
    case KIND_GENERIC:
      n += snprintf(tmp + n, sizeof(tmp) - n, "kind=generic N=%lld batch=%lld sign=%d radices=", (long long)p->N,
                    (long long)p->batch, p->sign);
      rad(p->gs.R, p->gs.S);
      n += snprintf(tmp + n, sizeof(tmp) - n, " launches=1");
      break;
    case KIND_FOURSTEP:
      n += snprintf(tmp + n, sizeof(tmp) - n, "kind=fourstep N=%lld batch=%lld sign=%d M=%lld K=%lld cols=",
                    (long long)p->N, (long long)p->batch, p->sign, (long long)p->M, (long long)p->K);
      rad(p->ce->R, p->ce->S);
      n += snprintf(tmp + n, sizeof(tmp) - n, " rows=");
      rad(p->re->R, p->re->S);
      n += snprintf(tmp + n, sizeof(tmp) - n, " col_kernel=%s row_kernel=%s workspace=%lld launches=2", p->ce->name,
                    p->re->name, (long long)(p->N * p->batch * (int64_t)sizeof(float2)));
      break;
    case KIND_DIST:
      n += dist_describe(p->dist, tmp + n, sizeof(tmp) - n);
      break;
    case KIND_CLUSTER:
      n += snprintf(tmp + n, sizeof(tmp) - n,
                    "kind=cluster N=%lld batch=%lld sign=%d split=256x256 kernel=k_c16(cluster of 8 CTAs, DSMEM row "
                    "exchange, one HBM round trip) launches=1",
                    (long long)p->N, (long long)p->batch, p->sign);
      break;
    case KIND_DIRECT:
      n += snprintf(tmp + n, sizeof(tmp) - n,
                    "kind=direct N=%lld batch=%lld sign=%d kernel=k_direct_tc(tcgen05.mma kind::tf32, 3xTF32, "
                    "M=128 N=K=%lld) launches=1",
                    (long long)p->N, (long long)p->batch, p->sign, (long long)(2 * p->N));
      break;
    case KIND_JIT:
      n += snprintf(tmp + n, sizeof(tmp) - n, "kind=jit N=%lld batch=%lld sign=%d radices=", (long long)p->N,
                    (long long)p->batch, p->sign);
      rad(p->jit_R, p->jit_S);
      n += snprintf(tmp + n, sizeof(tmp) - n, " kernel=fftc_jit(nvrtc sm_100a) fpb=%d smem=%zu launches=1", p->jk->fpb,
                    p->jk->smem);
      break;
    case KIND_GPASS:
      n += snprintf(tmp + n, sizeof(tmp) - n, "kind=gpass N=%lld batch=%lld sign=%d passes=", (long long)p->N,
                    (long long)p->batch, p->sign);
      for (int s = 0; s < p->gp.p; ++s) {
        n += snprintf(tmp + n, sizeof(tmp) - n, "%s%d(", s ? "," : "", p->gp.st[s].L);
        rad(p->gp.st[s].R, p->gp.st[s].S);
        n += snprintf(tmp + n, sizeof(tmp) - n, ")%s", p->gp.st[s].jk ? "jit" : "");
      }
      n += snprintf(tmp + n, sizeof(tmp) - n, " workspace=%lld launches=%d",
                    (long long)(p->gp.p > 1 ? p->N * p->batch * (int64_t)sizeof(float2) : 0), p->gp.p);
      break;
    case KIND_L2:
      n += snprintf(tmp + n, sizeof(tmp) - n, "kind=l2 N=%lld batch=%lld sign=%d passes=", (long long)p->N,
                    (long long)p->batch, p->sign);
      for (int s = 0; s < p->l2.p; ++s) n += snprintf(tmp + n, sizeof(tmp) - n, "%s%d", s ? "x" : "", p->l2.L[s]);
      n += snprintf(tmp + n, sizeof(tmp) - n, " kernel=%s chunk=%d ring_slots=%d lag=%d workspace=%lld launches=1",
                    p->l2.e->name, p->l2.tc, p->l2.slots, p->l2.lag, (long long)l2_work_bytes(p->l2, p->batch));
      break;
    case KIND_PASSES:
      n += snprintf(tmp + n, sizeof(tmp) - n, "kind=passes N=%lld batch=%lld sign=%d passes=", (long long)p->N,
                    (long long)p->batch, p->sign);
      for (int s = 0; s < p->pp.p; ++s) n += snprintf(tmp + n, sizeof(tmp) - n, "%s%s", s ? "," : "", p->pp.e[s]->name);
      n += snprintf(tmp + n, sizeof(tmp) - n, " tile_groups=");
      for (int s = 0; s < p->pp.p; ++s) n += snprintf(tmp + n, sizeof(tmp) - n, "%s%d", s ? "," : "", p->pp.group[s]);
      n += snprintf(tmp + n, sizeof(tmp) - n, " tma=tensor3d/4d workspace=%lld launches=%d",
                    (long long)(p->N * p->batch * (int64_t)sizeof(float2)), p->pp.p);
      break;
  }
  if (buf && len) {
    strncpy(buf, tmp, len - 1);
    buf[len - 1] = 0;
  }
  return n;
}

int fftc_candidates(int64_t N, const char** names, int max) {
  int c = 0;
  for (int i = 0; i < fused_count(); ++i)
    if (fused_at(i)->N == N) {
      if (names && c < max) names[c] = fused_at(i)->name;
      ++c;
    }
  return c;
}

int fftc_factorize(int64_t N, int* radices, int max) { return single_pass_radices(N, radices, max); }

int fftc_plan_split(int64_t N, int64_t* M, int64_t* K) { return top_split(N, M, K); }

int fftc_plan_passes(int64_t N, int* lengths, int max) { return pass_split(N, lengths, max); }

int fftc_plan_gpasses(int64_t N, int* lengths, int max) {
  // as the plan does: JIT passes up to 512 long when NVRTC is there, else the compiled 256
  const char* ej = getenv("FFTC_GPASS_JIT");
  const bool jit = jit_available() && !(ej && strcmp(ej, "0") == 0);
  return gpass_split(N, lengths, max, 7, jit ? kGpassSplitMaxL : kGpassMaxL);
}

int fftc_expr_radices(const char* expr, int64_t* N, int* radices, int max, char* err, size_t errlen) {
  int64_t r[64];
  const int S = expr_radices(expr, N, r, 64, err, errlen);
  if (S < 0) return -1;
  if (S > max) {
    if (err && errlen) snprintf(err, errlen, "more than %d stages", max);
    return -1;
  }
  for (int s = 0; s < S; ++s) {
    if (r[s] > 0x7fffffff) {
      if (err && errlen) snprintf(err, errlen, "radix too large");
      return -1;
    }
    if (radices) radices[s] = (int)r[s];
  }
  return S;
}

fftc_plan* fftc_plan_create_radices(int64_t N, int64_t batch, int sign, const int* radices, int S) {
  g_last = FFTC_SUCCESS;
  if (N < 1 || batch < 0 || (sign != -1 && sign != 1) || S < 0 || S > kMaxStages || (S > 0 && !radices))
    return fail(nullptr, FFTC_ERROR_INVALID_VALUE);
  if (S == 0) return fftc_plan_create(N, batch, sign);
  int64_t prod = 1;
  for (int s = 0; s < S; ++s) {
    if (radices[s] < 2) return fail(nullptr, FFTC_ERROR_INVALID_VALUE);
    prod *= radices[s];
    if (prod > N) return fail(nullptr, FFTC_ERROR_INVALID_VALUE);
  }
  if (prod != N) return fail(nullptr, FFTC_ERROR_INVALID_VALUE);
  if (!seven_smooth(N)) return fail(nullptr, FFTC_ERROR_UNSUPPORTED_SIZE);
  if (batch > 0 && batch > ((int64_t)1 << 60) / (N * 8)) return fail(nullptr, FFTC_ERROR_UNSUPPORTED_SIZE);
  int dev = 0;
  fftc_status ds = fftc_check_device(&dev);
  if (ds != FFTC_SUCCESS) return fail(nullptr, ds);
  fftc_plan* p = new fftc_plan();
  p->N = N;
  p->batch = batch;
  p->sign = sign;
  p->device = dev;
  cudaError_t err = cudaSuccess;
  if (N <= kGenericMaxN) {
    // a compiled schedule with exactly these stages, else the runtime-schedule kernel
    for (int i = 0; i < fused_count(); ++i) {
      const FusedEntry* e = fused_at(i);
      if (e->N != N || e->S != S) continue;
      bool same = true;
      for (int s = 0; s < S; ++s) same = same && e->R[s] == radices[s];
      if (!same) continue;
      p->kind = KIND_FUSED;
      p->fe = e;
      p->d_tw = upload_stage_table(N, e->R, e->S, &err);
      return err == cudaSuccess ? p : fail(p, from_cuda(err));
    }
    // no compiled schedule with exactly these stages: a kernel generated for them (NVRTC), else
    // the runtime-schedule kernel
    const char* sj = getenv("FFTC_SMOOTH_JIT");
    if (jit_available() && !(sj && strcmp(sj, "0") == 0) && S <= 32) {
      p->jk = jit_get_r((int)N, radices, S, &err);
      if (p->jk) {
        p->kind = KIND_JIT;
        p->jit_S = S;
        for (int s = 0; s < S; ++s) p->jit_R[s] = radices[s];
        p->d_tw = upload_stage_table(N, radices, S, &err);
        return err == cudaSuccess ? p : fail(p, from_cuda(err));
      }
      err = cudaSuccess;
    }
    for (int s = 0; s < S; ++s)
      if (!generic_supports_radix(radices[s])) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
    p->kind = KIND_GENERIC;
    p->gs.N = (int)N;
    p->gs.S = S;
    for (int s = 0; s < S; ++s) p->gs.R[s] = radices[s];
    p->d_tw = upload_stage_table(N, radices, S, &err);
    return err == cudaSuccess ? p : fail(p, from_cuda(err));
  }
  // above the single-pass limit: consecutive stages grouped into passes of <= kGpassMaxL
  int Lg[kMaxGPasses], R[kMaxGPasses][kMaxStages], Sg[kMaxGPasses];
  int pg = 0;
  int64_t cur = 1;
  for (int s = 0; s < S; ++s) {
    if (radices[s] > kGpassMaxL) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
    if (pg == 0 || cur * radices[s] > kGpassMaxL) {
      if (pg == kMaxGPasses) return fail(p, FFTC_ERROR_UNSUPPORTED_SIZE);
      Sg[pg] = 0;
      Lg[pg] = 1;
      cur = 1;
      ++pg;
    }
    R[pg - 1][Sg[pg - 1]++] = radices[s];
    Lg[pg - 1] *= radices[s];
    cur *= radices[s];
  }
  const fftc_status st = setup_gpass(p, Lg, pg, R, Sg);
  return st == FFTC_SUCCESS ? p : fail(p, st);
}

fftc_plan* fftc_plan_create_direct(int64_t N, int64_t batch, int sign) {
  g_last = FFTC_SUCCESS;
  if (N < 1 || batch < 0 || (sign != -1 && sign != 1)) return fail(nullptr, FFTC_ERROR_INVALID_VALUE);
  if (!direct_supported(N)) return fail(nullptr, FFTC_ERROR_UNSUPPORTED_SIZE);
  if (batch > 0 && batch > ((int64_t)1 << 60) / (N * 8)) return fail(nullptr, FFTC_ERROR_UNSUPPORTED_SIZE);
  int dev = 0;
  fftc_status ds = fftc_check_device(&dev);
  if (ds != FFTC_SUCCESS) return fail(nullptr, ds);
  fftc_plan* p = new fftc_plan();
  p->N = N;
  p->batch = batch;
  p->sign = sign;
  p->device = dev;
  p->kind = KIND_DIRECT;
  cudaError_t err = cudaSuccess;
  p->d_direct = direct_tables(N, sign, &err);
  if (err != cudaSuccess) return fail(p, from_cuda(err));
  return p;
}

int fftc_jit_source(int64_t N, char* buf, size_t len) {
  if (N < 2 || N > kGenericMaxN) return -1;
  const std::string src = jit_source((int)N);
  if (src.empty()) return -1;
  if (buf && len) {
    strncpy(buf, src.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return (int)src.size();
}

int fftc_jit_codelet_source(int R, char* buf, size_t len) {
  const std::string src = jit_codelet_source(R);
  if (src.empty()) return -1;
  if (buf && len) {
    strncpy(buf, src.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return (int)src.size();
}

int fftc_jit_compile(int64_t N, char* log, size_t loglen) {
  if (N < 2 || N > kGenericMaxN) return -1;
  std::string cubin, lg;
  const int rc = jit_compile_cubin((int)N, &cubin, &lg);
  if (log && loglen) {
    strncpy(log, lg.c_str(), loglen - 1);
    log[loglen - 1] = 0;
  }
  return rc == 0 ? (int)cubin.size() : rc;
}

int fftc_jit_pass_source(int L, char* buf, size_t len) {
  int R[32];
  const int S = jit_pass_radices(L, R, 32);
  if (L < 2 || L > kJitPassMaxL || S < 1) return -1;
  const std::string src = jit_pass_source(L, R, S);
  if (buf && len) {
    strncpy(buf, src.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return (int)src.size();
}

int fftc_jit_pass_compile(int L, char* log, size_t loglen) {
  int R[32];
  const int S = jit_pass_radices(L, R, 32);
  if (L < 2 || L > kJitPassMaxL || S < 1) return -1;
  std::string cubin, lg;
  const int rc = jit_compile_src_public(jit_pass_source(L, R, S), &cubin, &lg);
  if (log && loglen) {
    strncpy(log, lg.c_str(), loglen - 1);
    log[loglen - 1] = 0;
  }
  return rc == 0 ? (int)cubin.size() : rc;
}

fftc_plan* fftc_plan_create_expr(const char* expr, int64_t batch, int sign) {
  int64_t N = 0;
  int R[kMaxStages];
  const int S = fftc_expr_radices(expr, &N, R, kMaxStages, nullptr, 0);
  if (S < 0) return fail(nullptr, FFTC_ERROR_INVALID_VALUE);
  return fftc_plan_create_radices(N, batch, sign, R, S);
}

}  // extern "C"
