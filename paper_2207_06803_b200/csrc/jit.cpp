// jit.cpp -- JIT-compiled codelets for N with prime factors > 7 (product path, host side).
//
// The paper distinguishes a JIT mode, in which the transform size is a runtime value and
// the code is generated and compiled when it is requested, from an AOT mode with the size
// fixed at compile time, and names FFTW-style generated codelets as the
// way to go beyond its dense matrices.  The AOT side here is the set of
// compiled schedules (kernels_*.cu, passes.cu); this file is the JIT side: for an N <= 4096
// whose prime factors go beyond the compiled codelet set {2, 3, 5, 7} (primes up to
// kJitMaxPrime), it generates a single-pass Stockham kernel specialised to N -- every
// stage one level of Eq. 2, every DFT_R a straight-line codelet emitted by the
// same recursion (R = K M: K M-point codelets on the stride-K sub-vectors, constant
// twiddles w_R^{rj}, M K-point codelets; a prime R in the conjugate-pair symmetric form
// of the definition) -- compiles it with NVRTC for sm_100a and loads it through
// the driver API.  Kernels are cached per N for the life of the process.
//
// No link-time dependency: libnvrtc is dlopen'ed on first use and the driver entry points
// come from cudaGetDriverEntryPoint, so the library still loads where neither exists.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "jit.h"

namespace fftc {

namespace {

// ---------------------------------------------------------------- source generation
struct Emitter {
  std::string src;
  int tmp = 0;
  std::string fresh() { return "t" + std::to_string(tmp++); }
  void line(const std::string& l) { src += "  " + l + "\n"; }
};

std::string flit(double v) {
  char b[48];
  snprintf(b, sizeof b, "%.9ef", v);
  return b;
}

int smallest_prime(int n) {
  for (int p = 2; p * p <= n; ++p)
    if (n % p == 0) return p;
  return n;
}

// name = a * w_R^e, w_R = exp(-2 pi i / R); trivial angles resolved
std::string emit_twiddle(Emitter& E, const std::string& a, long long e, int R) {
  e %= R;
  if (e < 0) e += R;
  if (e == 0) return a;
  const std::string t = E.fresh();
  if ((8 * e) % R == 0) {
    const int k8 = (int)((8 * e) / R);  // angle -k8 pi / 4
    const std::string h = "0.70710678118654752f";
    switch (k8) {
      case 2: E.line("const cf " + t + " = cf{" + a + ".y, -" + a + ".x};"); break;
      case 4: E.line("const cf " + t + " = cf{-" + a + ".x, -" + a + ".y};"); break;
      case 6: E.line("const cf " + t + " = cf{-" + a + ".y, " + a + ".x};"); break;
      case 1: E.line("const cf " + t + " = cf{(" + a + ".x + " + a + ".y) * " + h + ", (" + a + ".y - " + a + ".x) * " + h + "};"); break;
      case 3: E.line("const cf " + t + " = cf{(" + a + ".y - " + a + ".x) * " + h + ", -(" + a + ".x + " + a + ".y) * " + h + "};"); break;
      case 5: E.line("const cf " + t + " = cf{-(" + a + ".x + " + a + ".y) * " + h + ", (" + a + ".x - " + a + ".y) * " + h + "};"); break;
      default: E.line("const cf " + t + " = cf{(" + a + ".x - " + a + ".y) * " + h + ", (" + a + ".x + " + a + ".y) * " + h + "};"); break;
    }
    return t;
  }
  const double ang = 2.0 * M_PI * (double)e / (double)R;
  const std::string c = flit(cos(ang)), s = flit(-sin(ang));
  E.line("const cf " + t + " = cf{fmaf(" + a + ".x, " + c + ", -" + a + ".y * " + s + "), fmaf(" + a + ".x, " + s +
         ", " + a + ".y * " + c + ")};");
  return t;
}

// y = DFT_R x (forward), straight-line; returns the output variable names.
std::vector<std::string> emit_dft(Emitter& E, const std::vector<std::string>& x) {
  const int R = (int)x.size();
  if (R == 1) return x;
  if (R == 2) {
    const std::string a = E.fresh(), b = E.fresh();
    E.line("const cf " + a + " = cf{" + x[0] + ".x + " + x[1] + ".x, " + x[0] + ".y + " + x[1] + ".y};");
    E.line("const cf " + b + " = cf{" + x[0] + ".x - " + x[1] + ".x, " + x[0] + ".y - " + x[1] + ".y};");
    return {a, b};
  }
  const int p = smallest_prime(R);
  if (p == R) {
    // prime: conjugate-pair symmetric form of y_k = sum_n x_n w^{nk}
    const int h = (R - 1) / 2;
    std::vector<std::string> s(h + 1), d(h + 1);
    for (int j = 1; j <= h; ++j) {
      s[j] = E.fresh();
      d[j] = E.fresh();
      E.line("const cf " + s[j] + " = cf{" + x[j] + ".x + " + x[R - j] + ".x, " + x[j] + ".y + " + x[R - j] + ".y};");
      E.line("const cf " + d[j] + " = cf{" + x[j] + ".x - " + x[R - j] + ".x, " + x[j] + ".y - " + x[R - j] + ".y};");
    }
    std::vector<std::string> y(R);
    y[0] = E.fresh();
    {
      std::string ex = x[0] + ".x", ey = x[0] + ".y";
      for (int j = 1; j <= h; ++j) {
        ex += " + " + s[j] + ".x";
        ey += " + " + s[j] + ".y";
      }
      E.line("const cf " + y[0] + " = cf{" + ex + ", " + ey + "};");
    }
    for (int k = 1; k <= h; ++k) {
      const std::string A = E.fresh(), B = E.fresh();
      std::string ax = x[0] + ".x", ay = x[0] + ".y", bx = "0.f", by = "0.f";
      for (int j = 1; j <= h; ++j) {
        const double th = 2.0 * M_PI * (double)((long long)j * k % R) / (double)R;
        ax = "fmaf(" + s[j] + ".x, " + flit(cos(th)) + ", " + ax + ")";
        ay = "fmaf(" + s[j] + ".y, " + flit(cos(th)) + ", " + ay + ")";
        bx = "fmaf(" + d[j] + ".x, " + flit(sin(th)) + ", " + bx + ")";
        by = "fmaf(" + d[j] + ".y, " + flit(sin(th)) + ", " + by + ")";
      }
      E.line("const cf " + A + " = cf{" + ax + ", " + ay + "};");
      y[k] = E.fresh();
      y[R - k] = E.fresh();
      if (h == 1) {
        // R = 3: the single sine term folded into the outputs (one FMA per component, as the
        // compiled Codelet<3>)
        const std::string sn = flit(sin(2.0 * M_PI * (double)k / (double)R));
        E.line("const cf " + y[k] + " = cf{fmaf(" + d[1] + ".y, " + sn + ", " + A + ".x), fmaf(" + d[1] + ".x, -" + sn +
               ", " + A + ".y)};");
        E.line("const cf " + y[R - k] + " = cf{fmaf(" + d[1] + ".y, -" + sn + ", " + A + ".x), fmaf(" + d[1] + ".x, " +
               sn + ", " + A + ".y)};");
        continue;
      }
      E.line("const cf " + B + " = cf{" + bx + ", " + by + "};");
      // y_k = A - i B, y_{R-k} = A + i B
      E.line("const cf " + y[k] + " = cf{" + A + ".x + " + B + ".y, " + A + ".y - " + B + ".x};");
      E.line("const cf " + y[R - k] + " = cf{" + A + ".x - " + B + ".y, " + A + ".y + " + B + ".x};");
    }
    return y;
  }
  const int K = (R % 4 == 0 && R > 4) ? 4 : p, M = R / K;
  int g = K, h = M;
  while (h) {
    const int t = g % h;
    g = h;
    h = t;
  }
  if (g == 1) {
    // coprime K, M: Good-Thomas prime-factor form of the same DFT_R (DESIGN reading 19) --
    // n = (n1 M + n2 K) mod R, k = (k1 eK + k2 eM) mod R with eK = 1 mod K, 0 mod M and
    // eM = 0 mod K, 1 mod M; no internal twiddles
    int eK = 0, eM = 0;
    for (int t = 0; t < R; ++t) {
      if (t % K == 1 % K && t % M == 0) eK = t;
      if (t % K == 0 && t % M == 1 % M) eM = t;
    }
    std::vector<std::vector<std::string>> z((size_t)K);
    for (int n1 = 0; n1 < K; ++n1) {
      std::vector<std::string> sub((size_t)M);
      for (int n2 = 0; n2 < M; ++n2) sub[n2] = x[(size_t)((n1 * M + n2 * K) % R)];
      z[n1] = emit_dft(E, sub);
    }
    std::vector<std::string> y((size_t)R);
    for (int k2 = 0; k2 < M; ++k2) {
      std::vector<std::string> col((size_t)K);
      for (int n1 = 0; n1 < K; ++n1) col[n1] = z[n1][k2];
      const std::vector<std::string> o = emit_dft(E, col);
      for (int k1 = 0; k1 < K; ++k1) y[(size_t)((k1 * eK + k2 * eM) % R)] = o[k1];
    }
    return y;
  }
  // composite R = K M, Eq. 2: (DFT_K (x) I_M) D^R_M (I_K (x) DFT_M) Pi^R_K
  std::vector<std::vector<std::string>> z((size_t)K);
  for (int r = 0; r < K; ++r) {
    std::vector<std::string> sub((size_t)M);
    for (int q = 0; q < M; ++q) sub[q] = x[(size_t)q * K + r];  // Pi^R_K
    z[r] = emit_dft(E, sub);                                     // I_K (x) DFT_M
    for (int j = 0; j < M; ++j) z[r][j] = emit_twiddle(E, z[r][j], (long long)r * j, R);  // D^R_M
  }
  std::vector<std::string> y((size_t)R);
  for (int j = 0; j < M; ++j) {
    std::vector<std::string> col((size_t)K);
    for (int r = 0; r < K; ++r) col[r] = z[r][j];
    const std::vector<std::string> o = emit_dft(E, col);  // DFT_K (x) I_M
    for (int k1 = 0; k1 < K; ++k1) y[(size_t)j + (size_t)M * k1] = o[k1];
  }
  return y;
}

std::string codelet_fn(int R) {
  Emitter E;
  std::vector<std::string> x((size_t)R);
  for (int r = 0; r < R; ++r) {
    x[r] = "x" + std::to_string(r);
    E.line("const cf " + x[r] + " = v[" + std::to_string(r) + "];");
  }
  const std::vector<std::string> y = emit_dft(E, x);
  for (int r = 0; r < R; ++r) E.line("v[" + std::to_string(r) + "] = " + y[r] + ";");
  return "__device__ __forceinline__ void dft" + std::to_string(R) + "(cf* v) {\n" + E.src + "}\n";
}

}  // namespace

std::string jit_codelet_source(int R) { return (R >= 2 && R <= 128) ? codelet_fn(R) : std::string(); }

int jit_radices(int N, int* R, int max) {
  if (N < 2) return -1;
  std::vector<int> out;
  int n = N;
  int a = 0;
  while (n % 2 == 0) {
    n /= 2;
    ++a;
  }
  for (int i = 0; i < a / 4; ++i) out.push_back(16);
  if (a % 4) out.push_back(1 << (a % 4));
  while (n % 9 == 0) {
    out.push_back(9);
    n /= 9;
  }
  if (n % 3 == 0) {
    out.push_back(3);
    n /= 3;
  }
  while (n % 25 == 0) {
    out.push_back(25);
    n /= 25;
  }
  if (n % 5 == 0) {
    out.push_back(5);
    n /= 5;
  }
  while (n % 7 == 0) {
    out.push_back(7);
    n /= 7;
  }
  for (int p = 11; n > 1; p += 2) {
    if (p > kJitMaxPrime) return -1;
    while (n % p == 0) {
      out.push_back(p);
      n /= p;
    }
  }
  if ((int)out.size() > max) return -1;
  for (size_t i = 0; i < out.size(); ++i) R[i] = out[i];
  return (int)out.size();
}

int jit_pass_radices(int L, int* R, int max) {
  std::vector<int> f;
  int n = L;
  for (int p = 2; p <= n; ++p)
    while (n % p == 0) {
      if (p > kJitMaxPrime) return -1;
      f.push_back(p);
      n /= p;
    }
  // balanced groups (fewest stages with every radix <= 32, or a lone prime): more butterflies
  // per stage than peeling 16s/25s off, e.g. 100 -> 10 x 10 instead of 4 x 25
  for (int g = 1; g <= 4; ++g) {
    std::vector<int> grp((size_t)g, 1);
    for (size_t i = f.size(); i-- > 0;) {  // largest primes first, onto the smallest group
      size_t best = 0;
      for (size_t j = 1; j < grp.size(); ++j)
        if (grp[j] < grp[best]) best = j;
      grp[best] *= f[i];
    }
    bool ok = true;
    for (int x : grp) ok = ok && (x <= 32 || (x <= kJitMaxPrime && smallest_prime(x) == x));
    if (!ok && g < 4) continue;
    if (g > max) return -1;
    int S = 0;
    for (int x : grp)
      if (x > 1) R[S++] = x;
    return S;
  }
  return -1;
}

int jit_fpb(int N) {
  int f = kJitTile / N;
  return f < 1 ? 1 : f;
}

namespace {

// Stockham sub-stages of DFT_L over `count` rows (transforms / columns) held at pitch P in
// shared memory, ping-ponging between A and B (one level of Eq. 2 per stage); twiddles from
// the stage table `tw` (entry (Ns-1) + (r-1) Ns + m = w^{m r}).
void emit_stages(std::string& s, int L, const int* R, int S, const char* count, int P) {
  char b[640];
  int Ns = 1;
  for (int i = 0; i < S; ++i) {
    const int Rs = R[i], NB = L / Rs;
    snprintf(b, sizeof b,
             "  { // sub-stage %d: radix %d, Ns %d\n"
             "    for (int q = threadIdx.x; q < (%s) * %d; q += T) {\n"
             "      const int f = q / %d, j = q %% %d, m = j %% %d;\n"
             "      const cf* a = A + f * %d; cf* bb = B + f * %d;\n"
             "      cf v[%d];\n"
             "      for (int r = 0; r < %d; ++r) v[r] = a[j + r * %d];\n",
             i, Rs, Ns, count, NB, NB, NB, Ns, P, P, Rs, Rs, NB);
    s += b;
    if (Ns > 1) {
      snprintf(b, sizeof b,
               "      for (int r = 1; r < %d; ++r) { const cf w = tw[%d + (r - 1) * %d + m];\n"
               "        v[r] = cf{fmaf(v[r].x, w.x, -v[r].y * w.y), fmaf(v[r].x, w.y, v[r].y * w.x)}; }\n",
               Rs, Ns - 1, Ns);
      s += b;
    }
    snprintf(b, sizeof b,
             "      dft%d(v);\n"
             "      const int o = (j / %d) * %d + m;\n"
             "      for (int r = 0; r < %d; ++r) bb[o + r * %d] = v[r];\n"
             "    }\n"
             "    __syncthreads(); cf* t = A; A = B; B = t;\n"
             "  }\n",
             Rs, Ns, Ns * Rs, Rs, Ns);
    s += b;
    Ns *= Rs;
  }
}

// In-place variant for long passes (one buffer, half the shared memory): every thread first
// reads all of its butterflies of the stage into registers (KB = ceil(COLS NB / T) per thread,
// compile-time), the CTA syncs, then writes -- as the compiled fused kernels do.
void emit_stages_inplace(std::string& s, int L, const int* R, int S, int COLS, int T, int P) {
  char b[900];
  int Ns = 1;
  for (int i = 0; i < S; ++i) {
    const int Rs = R[i], NB = L / Rs, KB = (COLS * NB + T - 1) / T;
    snprintf(b, sizeof b,
             "  { // sub-stage %d (in place): radix %d, Ns %d\n"
             "    cf v[%d][%d]; int jj[%d], ff[%d];\n"
             "#pragma unroll\n"
             "    for (int kb = 0; kb < %d; ++kb) { const int q = threadIdx.x + kb * T; ff[kb] = -1;\n"
             "      if (q < nc * %d) { const int f = q / %d, j = q %% %d; ff[kb] = f; jj[kb] = j;\n"
             "#pragma unroll\n"
             "        for (int r = 0; r < %d; ++r) v[kb][r] = A[f * %d + j + r * %d]; } }\n"
             "    __syncthreads();\n"
             "#pragma unroll\n"
             "    for (int kb = 0; kb < %d; ++kb) { if (ff[kb] < 0) continue; const int f = ff[kb], j = jj[kb], m = j %% %d;\n",
             i, Rs, Ns, KB, Rs, KB, KB, KB, NB, NB, NB, Rs, P, NB, KB, Ns);
    s += b;
    if (Ns > 1) {
      snprintf(b, sizeof b,
               "#pragma unroll\n"
               "      for (int r = 1; r < %d; ++r) { const cf w = tw[%d + (r - 1) * %d + m];\n"
               "        v[kb][r] = cf{fmaf(v[kb][r].x, w.x, -v[kb][r].y * w.y), fmaf(v[kb][r].x, w.y, v[kb][r].y * w.x)}; }\n",
               Rs, Ns - 1, Ns);
      s += b;
    }
    snprintf(b, sizeof b,
             "      dft%d(v[kb]);\n"
             "      const int o = (j / %d) * %d + m;\n"
             "#pragma unroll\n"
             "      for (int r = 0; r < %d; ++r) A[f * %d + o + r * %d] = v[kb][r];\n"
             "    }\n"
             "    __syncthreads();\n"
             "  }\n",
             Rs, Ns, Ns * Rs, Rs, P, Ns);
    s += b;
    Ns *= Rs;
  }
}

std::string prelude(const int* R, int S) {
  std::string s = "struct alignas(8) cf { float x, y; };\n";
  std::vector<int> done;
  for (int i = 0; i < S; ++i) {
    bool seen = false;
    for (int d : done) seen = seen || d == R[i];
    if (seen) continue;
    done.push_back(R[i]);
    s += codelet_fn(R[i]);
  }
  return s;
}

}  // namespace

std::string jit_source(int N) {
  int R[32];
  const int S = jit_radices(N, R, 32);
  if (S < 0) return "";
  const int FPB = jit_fpb(N), NP = N | 1;
  std::string s = "// generated by libfftc (jit.cpp) for N = " + std::to_string(N) + "\n" + prelude(R, S);
  char b[512];
  snprintf(b, sizeof b,
           "extern \"C\" __global__ void __launch_bounds__(%d) fftc_jit(const cf* __restrict__ in, cf* __restrict__ out,\n"
           "    const cf* __restrict__ tw, long long batch, float csign) {\n"
           "  extern __shared__ cf sm[];\n"
           "  constexpr int N = %d, FPB = %d, NP = %d, T = %d;\n",
           kJitThreads, N, FPB, NP, kJitThreads);
  s += b;
  s += "  const long long f0 = (long long)blockIdx.x * FPB;\n"
       "  const int nf = (int)(batch - f0 < FPB ? batch - f0 : FPB);\n"
       "  cf* A = sm; cf* B = sm + FPB * NP;\n"
       "  const cf* gi = in + f0 * N; cf* go = out + f0 * N;\n"
       "  for (int e = threadIdx.x; e < nf * N; e += T) { const cf a = gi[e]; A[(e / N) * NP + e % N] = cf{a.x, csign * a.y}; }\n"
       "  __syncthreads();\n";
  emit_stages(s, N, R, S, "nf", NP);
  s += "  for (int e = threadIdx.x; e < nf * N; e += T) { const cf a = A[(e / N) * NP + e % N]; go[e] = cf{a.x, csign * a.y}; }\n"
       "}\n";
  return s;
}

int jit_pass_cols(int L) {
  if (L > 256) return 8;  // long passes: in place, 8 columns (64-byte rows), <= 66 KB
  int c = 16;
  while (c < 256 && 2 * c * L <= 4096) c *= 2;
  return c;
}
size_t jit_pass_smem(int L) {
  return (size_t)(L > 256 ? 1 : 2) * jit_pass_cols(L) * (L + 1) * 8;
}

// One pass of the runtime multi-pass path (the kernel of gpass.cu) with L, its radices and
// the column count compiled in: straight-line codelets (any prime up to kJitMaxPrime),
// constant-divisor index math.  Ns, the twiddle split and the sizes stay runtime arguments,
// so one kernel serves every pass of that length.
std::string jit_pass_source(int L, const int* R, int S) {
  const int LP = L + 1, COLS = jit_pass_cols(L);
  int LC = 0;
  while ((1 << LC) < COLS) ++LC;
  std::string s = "// generated by libfftc (jit.cpp): pass of length " + std::to_string(L) + "\n" + prelude(R, S);
  char b[900];
  snprintf(b, sizeof b,
           "extern \"C\" __global__ void __launch_bounds__(%d, 4) fftc_jit_pass(const cf* __restrict__ in,\n"
           "    cf* __restrict__ out, const cf* __restrict__ tw, const cf* __restrict__ twA, const cf* __restrict__ twB,\n"
           "    long long N, int Ns, int tws, int tiles, float csign_in, float csign_out) {\n"
           "  extern __shared__ cf sm[];\n"
           "  constexpr int L = %d, LP = %d, COLS = %d, LC = %d, T = %d;\n"
           "  __shared__ int s_cq[COLS], s_cm[COLS];\n",
           kJitThreads, L, LP, COLS, LC, kJitThreads);
  s += b;
  s += "  const long long NB = N / L;\n"
       "  const long long bt = blockIdx.x / tiles;\n"
       "  const long long c0 = (long long)(blockIdx.x % tiles) * COLS;\n"
       "  const int nc = (int)(NB - c0 < COLS ? NB - c0 : COLS);\n"
       "  cf* A = sm;\n"
       "  for (int f = threadIdx.x; f < COLS; f += T) { const int c = (int)c0 + f; s_cq[f] = c / Ns; s_cm[f] = c - (c / Ns) * Ns; }\n"
       "  __syncthreads();\n"
       "  const cf* gi = in + bt * N + c0;\n"
       "  const long long amask = (1LL << tws) - 1;\n"
       "  for (int e0 = threadIdx.x; e0 < (L << LC); e0 += 8 * T) {\n"
       "    cf v[8];\n"
       "#pragma unroll\n"
       "    for (int u = 0; u < 8; ++u) { const int e = e0 + u * T, f = e & (COLS - 1), r = e >> LC;\n"
       "      v[u] = (e < (L << LC) && f < nc) ? gi[f + (long long)r * NB] : cf{0.f, 0.f}; }\n"
       "#pragma unroll\n"
       "    for (int u = 0; u < 8; ++u) { const int e = e0 + u * T, f = e & (COLS - 1), r = e >> LC;\n"
       "      if (e < (L << LC) && f < nc) { cf x = v[u]; x.y *= csign_in;\n"
       "        if (Ns > 1) { const long long ex = (long long)s_cm[f] * r;\n"
       "          const cf p = twA[ex & amask], q = twB[ex >> tws];\n"
       "          const cf w = cf{fmaf(p.x, q.x, -p.y * q.y), fmaf(p.x, q.y, p.y * q.x)};\n"
       "          x = cf{fmaf(x.x, w.x, -x.y * w.y), fmaf(x.x, w.y, x.y * w.x)}; }\n"
       "        A[f * LP + r] = x; } }\n"
       "  }\n"
       "  __syncthreads();\n";
  if (L > 256) {
    emit_stages_inplace(s, L, R, S, COLS, kJitThreads, LP);
  } else {
    s += "  cf* B = sm + COLS * LP;\n";
    emit_stages(s, L, R, S, "nc", LP);
  }
  s += "  cf* go = out + bt * N;\n"
       "  if (Ns == 1) {\n"
       "    for (int e = threadIdx.x; e < nc * L; e += T) { const int f = e / L, r = e - (e / L) * L;\n"
       "      const cf a = A[f * LP + r]; go[(c0 + f) * L + r] = cf{a.x, csign_out * a.y}; }\n"
       "  } else {\n"
       "    for (int e = threadIdx.x; e < (L << LC); e += T) { const int f = e & (COLS - 1), r = e >> LC;\n"
       "      if (f < nc) { const cf a = A[f * LP + r];\n"
       "        go[((long long)s_cq[f] * L + r) * Ns + s_cm[f]] = cf{a.x, csign_out * a.y}; } }\n"
       "  }\n"
       "}\n";
  return s;
}

// ---------------------------------------------------------------- NVRTC + driver API
namespace {

typedef int (*nvrtcCreateProgram_t)(void**, const char*, const char*, int, const char* const*, const char* const*);
typedef int (*nvrtcCompileProgram_t)(void*, int, const char* const*);
typedef int (*nvrtcGetSize_t)(void*, size_t*);
typedef int (*nvrtcGetData_t)(void*, char*);
typedef int (*nvrtcDestroyProgram_t)(void**);

struct Nvrtc {
  bool ok = false;
  nvrtcCreateProgram_t create = nullptr;
  nvrtcCompileProgram_t compile = nullptr;
  nvrtcGetSize_t log_size = nullptr, cubin_size = nullptr;
  nvrtcGetData_t log = nullptr, cubin = nullptr;
  nvrtcDestroyProgram_t destroy = nullptr;
};

const Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
      h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) return;
    n.create = (nvrtcCreateProgram_t)dlsym(h, "nvrtcCreateProgram");
    n.compile = (nvrtcCompileProgram_t)dlsym(h, "nvrtcCompileProgram");
    n.log_size = (nvrtcGetSize_t)dlsym(h, "nvrtcGetProgramLogSize");
    n.log = (nvrtcGetData_t)dlsym(h, "nvrtcGetProgramLog");
    n.cubin_size = (nvrtcGetSize_t)dlsym(h, "nvrtcGetCUBINSize");
    n.cubin = (nvrtcGetData_t)dlsym(h, "nvrtcGetCUBIN");
    n.destroy = (nvrtcDestroyProgram_t)dlsym(h, "nvrtcDestroyProgram");
    n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
  });
  return n;
}

template <class F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return (F)p;
}

std::mutex g_mu;
std::map<std::string, JitKernel*> g_cache;
std::string g_log;

int compile_src(const std::string& src, std::string* cubin, std::string* log) {
  const Nvrtc& n = nvrtc();
  if (!n.ok) return -1;
  if (src.empty()) return -2;
  void* prog = nullptr;
  if (n.create(&prog, src.c_str(), "fftc_jit.cu", 0, nullptr, nullptr) != 0) return -3;
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo"};
  const int rc = n.compile(prog, 3, opts);
  size_t ls = 0;
  n.log_size(prog, &ls);
  if (log) {
    log->assign(ls, '\0');
    if (ls) n.log(prog, &(*log)[0]);
  }
  if (rc != 0) {
    n.destroy(&prog);
    return -4;
  }
  size_t cs = 0;
  n.cubin_size(prog, &cs);
  cubin->assign(cs, '\0');
  n.cubin(prog, &(*cubin)[0]);
  n.destroy(&prog);
  return 0;
}

// Compile + load `src`, kernel `name`, dynamic shared memory `smem`; cached under `key`.
const JitKernel* load_kernel(const std::string& key, const std::string& src, const char* name, size_t smem, int N,
                             int fpb, cudaError_t* err) {
  std::lock_guard<std::mutex> lk(g_mu);
  // a loaded CUfunction belongs to the context (device) it was loaded in: cache per device
  int dev = 0;
  cudaGetDevice(&dev);
  const std::string dkey = key + "@" + std::to_string(dev);
  auto it = g_cache.find(dkey);
  if (it != g_cache.end()) {
    *err = cudaSuccess;
    return it->second;
  }
  typedef CUresult (*load_t)(CUmodule*, const void*);
  typedef CUresult (*getfn_t)(CUfunction*, CUmodule, const char*);
  typedef CUresult (*setattr_t)(CUfunction, CUfunction_attribute, int);
  static load_t load = driver_fn<load_t>("cuModuleLoadData");
  static getfn_t getfn = driver_fn<getfn_t>("cuModuleGetFunction");
  static setattr_t setattr = driver_fn<setattr_t>("cuFuncSetAttribute");
  *err = cudaErrorNotSupported;
  if (!load || !getfn || !setattr) return nullptr;
  // the driver-API module load needs the runtime's primary context to be current
  *err = cudaFree(nullptr);
  if (*err != cudaSuccess) return nullptr;
  *err = cudaErrorNotSupported;
  std::string cubin;
  if (compile_src(src, &cubin, &g_log) != 0) return nullptr;
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  if (load(&mod, cubin.data()) != CUDA_SUCCESS || getfn(&fn, mod, name) != CUDA_SUCCESS) {
    *err = cudaErrorInvalidKernelImage;
    return nullptr;
  }
  JitKernel* k = new JitKernel();
  k->fn = fn;
  k->N = N;
  k->fpb = fpb;
  k->smem = smem;
  if (setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)k->smem) != CUDA_SUCCESS) {
    delete k;
    *err = cudaErrorInvalidValue;
    return nullptr;
  }
  g_cache[dkey] = k;
  *err = cudaSuccess;
  return k;
}

}  // namespace

bool jit_available() { return nvrtc().ok; }

int jit_compile_cubin(int N, std::string* cubin, std::string* log) { return compile_src(jit_source(N), cubin, log); }

int jit_compile_src_public(const std::string& src, std::string* cubin, std::string* log) {
  return compile_src(src, cubin, log);
}

const JitKernel* jit_get(int N, cudaError_t* err) {
  const int fpb = jit_fpb(N);
  return load_kernel("n:" + std::to_string(N), jit_source(N), "fftc_jit", (size_t)2 * fpb * (N | 1) * 8, N, fpb, err);
}

const JitKernel* jit_pass_get(int L, const int* R, int S, cudaError_t* err) {
  std::string key = "p:" + std::to_string(L);
  for (int i = 0; i < S; ++i) key += ":" + std::to_string(R[i]);
  const int cols = jit_pass_cols(L);
  return load_kernel(key, jit_pass_source(L, R, S), "fftc_jit_pass", jit_pass_smem(L), L, cols, err);
}

cudaError_t jit_pass_launch(const JitKernel* k, const float2* in, float2* out, const float2* tw, const float2* twA,
                            const float2* twB, long long N, int Ns, int tws, long long batch, int conj_in,
                            int conj_out, cudaStream_t st) {
  typedef CUresult (*launch_t)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                               CUstream, void**, void**);
  static launch_t launch = driver_fn<launch_t>("cuLaunchKernel");
  if (!launch) return cudaErrorNotSupported;
  const long long NB = N / k->N;
  int tiles = (int)((NB + k->fpb - 1) / k->fpb);
  const long long grid = batch * tiles;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  float ci = conj_in ? -1.f : 1.f, co = conj_out ? -1.f : 1.f;
  void* args[] = {(void*)&in, (void*)&out, (void*)&tw, (void*)&twA, (void*)&twB, (void*)&N, (void*)&Ns,
                  (void*)&tws, (void*)&tiles, (void*)&ci, (void*)&co};
  const CUresult r = launch(k->fn, (unsigned)grid, 1, 1, kJitThreads, 1, 1, (unsigned)k->smem, (CUstream)st, args,
                            nullptr);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

cudaError_t jit_launch(const JitKernel* k, const float2* in, float2* out, const float2* tw, long long batch, int conj,
                       cudaStream_t st) {
  typedef CUresult (*launch_t)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                               CUstream, void**, void**);
  static launch_t launch = driver_fn<launch_t>("cuLaunchKernel");
  if (!launch) return cudaErrorNotSupported;
  const long long grid = (batch + k->fpb - 1) / k->fpb;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  float csign = conj ? -1.f : 1.f;
  void* args[] = {(void*)&in, (void*)&out, (void*)&tw, (void*)&batch, (void*)&csign};
  const CUresult r = launch(k->fn, (unsigned)grid, 1, 1, kJitThreads, 1, 1, (unsigned)k->smem, (CUstream)st, args,
                            nullptr);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

const char* jit_last_log() { return g_log.c_str(); }

}  // namespace fftc
