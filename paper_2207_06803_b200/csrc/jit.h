// jit.h -- JIT-compiled kernels for N with prime factors > 7 (product path, host side).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>

#include <string>

namespace fftc {

constexpr int kJitMaxPrime = 61;  // largest prime radix the JIT emits (conjugate-pair form, O(p^2))
constexpr int kJitThreads = 256;
constexpr int kJitTile = 4096;
constexpr int kJitLoadRound = 16;  // JIT pass kernels: rows loaded per thread per round    // elements per CTA (FPB = 4096 / N transforms)

struct JitKernel {
  CUfunction fn;
  // pass kernels: entry point per (first pass, conjugated input, conjugated output), index
  // first * 4 + ci * 2 + co (jit_pass_launch)
  static constexpr int kVariants = 8;
  CUfunction variant[kVariants] = {};
  int N, fpb;
  size_t smem;
  int threads = kJitThreads;  // CTA size (pass kernels choose theirs, jit_pass_geo)
};

// Tile geometry of a JIT pass kernel of length L (jit.cpp): columns per CTA, threads, pitch.
struct PassGeo {
  int cols = 0, threads = 0, lp = 0, minb = 1;
};
PassGeo jit_pass_geo(int L, const int* R, int S, int min_cols, bool single);  // rows per tile >= min_cols

// Radix schedule for the JIT kernel (16/8/4/2, 9/3, 25/5, 7, then primes 11..kJitMaxPrime),
// or -1 if N has a prime factor > kJitMaxPrime.
int jit_radices(int N, int* R, int max);
// Radices of a JIT pass kernel of length L: balanced groups of its prime factors.
int jit_pass_radices(int L, int* R, int max);
// The straight-line codelet dft<R>(cf* v) the emitter generates (2 <= R <= 128, else "").
std::string jit_codelet_source(int R);
// CUDA C++ source of the kernel specialised to N ("" if unsupported).
std::string jit_source(int N);
// ... for an explicit radix list R_0 (leaf) .. R_{S-1} (an FFTc expression's schedule)
std::string jit_source_r(int N, const int* R, int S);
// NVRTC compile to an sm_100a cubin (no device needed).  0 on success.
int jit_compile_cubin(int N, std::string* cubin, std::string* log);
int jit_compile_src_public(const std::string& src, std::string* cubin, std::string* log);
bool jit_available();
// Compiled + loaded kernel for N (cached per process).
const JitKernel* jit_get(int N, cudaError_t* err);
const JitKernel* jit_get_r(int N, const int* R, int S, cudaError_t* err);
cudaError_t jit_launch(const JitKernel* k, const float2* in, float2* out, const float2* tw, long long batch, int conj,
                       cudaStream_t st);
const char* jit_last_log();

// One pass of the runtime multi-pass path (gpass.cu) specialised to its length L and radices
// (any primes up to kJitMaxPrime), compiled by NVRTC and cached per (L, radices).
constexpr int kJitPassMaxL = 4096;  // longest JIT pass kernel (the fused variant, 2 columns, for 4096)
constexpr int kGpassSplitMaxL = 512;  // longest pass the default split uses (round 1: 1000-long passes were slower than three 100-long ones)
std::string jit_pass_source(int L, const int* R, int S);
const JitKernel* jit_pass_get(int L, const int* R, int S, cudaError_t* err);
cudaError_t jit_pass_launch(const JitKernel* k, const float2* in, float2* out, const float2* tw, const float2* twA,
                            const float2* twB, long long N, int Ns, int tws, long long batch, int conj_in,
                            int conj_out, cudaStream_t st);

}  // namespace fftc
