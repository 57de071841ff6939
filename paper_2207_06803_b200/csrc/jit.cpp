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

int jit_radices(int N, int* R, int max) {
  // the single-pass JIT kernel uses the pass kernels' balanced grouping (fewest stages with
  // every radix <= 32 or a lone prime: fewer barriers and less unrolled code than peeling
  // 16s, 9s, 25s and single primes off one at a time)
  if (N < 2) return -1;
  const int S = jit_pass_radices(N, R, max);
  // smallest radix as the leaf (measured on B200 with the generated kernel: 143 as 11 x 13
  // 0.26 ms vs 13 x 11 0.33 ms per 2^26 elements)
  for (int a = 1; a < S; ++a)
    for (int b = a; b > 0 && R[b] < R[b - 1]; --b) {
      const int t = R[b];
      R[b] = R[b - 1];
      R[b - 1] = t;
    }
  return S;
}



namespace {

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

namespace {
// replace every "$NAME" in t by its value
std::string subst(std::string t, const std::vector<std::pair<std::string, std::string>>& kv) {
  for (const auto& p : kv) {
    const std::string key = "$" + p.first;
    for (size_t at = t.find(key); at != std::string::npos; at = t.find(key, at + p.second.size()))
      t.replace(at, key.size(), p.second);
  }
  return t;
}
}  // namespace

// Geometry of a JIT pass kernel: COLS adjacent columns per CTA held in shared memory as
// [column][row] at an odd pitch LP (conflict-free both along rows and across columns), T threads.
// Chosen so that every sub-stage's COLS*L/R butterflies split evenly over the threads (no idle
// round), each thread's load/store column stays fixed (T a multiple of COLS), at most 48
// complex values per thread in registers, <= 100 KB of shared memory (>= 2 CTAs per SM), and
// the tile large enough to amortise the per-CTA work.
// Shared-memory layout of the generated kernels: row f, element i at f LP + i + i / P (macro SIDX).
// Single-pass kernels walk a transform's butterflies with consecutive lanes, so sub-stage 0 writes
// i = j R_0 + r at a lane stride of R_0 elements: when 4 | R_0 that is a 4- to 16-way bank
// conflict, and one pad element every P = R_0 (power of two) or 16 elements removes it.  Pass
// kernels load and store across columns (no such stride) and odd R_0 is conflict free: no padding
// (P = 0).  The row pitch LP >= L + L / P is odd (conflict free across rows).
int jit_padp(const int* R, bool single) {
  if (!single || R[0] % 4 != 0) return 0;
  return (R[0] & (R[0] - 1)) == 0 ? R[0] : 16;
}
int jit_pitch(int L, const int* R, bool single) {
  const int p = jit_padp(R, single);
  return (L + (p ? L / p : 0)) | 1;
}
std::string jit_sidx_macro(const int* R, bool single) {
  const int p = jit_padp(R, single);
  return p ? "#define SIDX(f, i) ((f) * LP + (i) + (i) / " + std::to_string(p) + ")\n"
           : std::string("#define SIDX(f, i) ((f) * LP + (i))\n");
}

PassGeo jit_pass_geo(int L, const int* R, int S, int min_cols, bool single) {
  PassGeo best;  // cols == 0: no feasible geometry (callers report UNSUPPORTED_SIZE)
  double bscore = -1.0;
  const int lp = jit_pitch(L, R, single);
  for (int cols = min_cols; cols <= 256; cols *= 2) {
    const size_t smem = (size_t)cols * lp * 8;
    if (smem > (size_t)100 * 1024) break;
    for (int T = 64; T <= 512; T += 32) {
      if (T % cols) continue;
      const int rstep = T / cols, E = (L + rstep - 1) / rstep;
      if (E > 64) continue;
      double useful = 0.0, slots = 0.0;
      int vals = E < kJitLoadRound ? E : kJitLoadRound;  // complex values live per thread
      bool ok = true;
      for (int q = 0; q < S; ++q) {
        const int nb = cols * (L / R[q]), kb = (nb + T - 1) / T;
        if (kb * R[q] > (R[q] > 32 ? R[q] : 32)) ok = false;  // one butterfly of a large prime is allowed
        if (kb * R[q] > vals) vals = kb * R[q];
        useful += (double)nb * R[q];
        slots += (double)kb * T * R[q];
      }
      if (!ok) continue;
      const double eff = (useful / slots) * ((double)L / ((double)E * rstep));
      const double tile = (double)cols * L;
      // resident CTAs per SM: registers (estimate: 2 per complex value + ~48 for addresses,
      // twiddles and codelet temporaries) and shared memory; at least two so one CTA's loads
      // and stores overlap another's compute
      const int regs = 2 * vals + 48;
      const int ctas_reg = 65536 / (T * (regs > 64 ? regs : 64));
      const int ctas_smem = (int)((227 * 1024) / (smem + 1024));
      const int ctas = ctas_reg < ctas_smem ? ctas_reg : ctas_smem;
      if (ctas < 1) continue;
      const double warps = (double)ctas * T / 32.0;
      // unrolled straight-line work per thread (values through every sub-stage): long kernels
      // thrash the instruction cache (a 2310-point kernel at ~100 values per thread measured
      // slower than the looped one it replaced)
      int work = 0;
      for (int q = 0; q < S; ++q) work += ((cols * (L / R[q]) + T - 1) / T) * R[q];
      const double score = eff + 0.03 * (tile < 4096 ? tile / 4096 : 1.0) + 0.06 * (warps < 24 ? warps / 24 : 1.0) +
                           (ctas >= 2 ? 0.1 : 0.0) - (work > 64 ? 0.002 * (work - 64) : 0.0);
      if (score > bscore + 1e-9) {
        bscore = score;
        best.cols = cols;
        best.threads = T;
        best.lp = lp;
        best.minb = ctas >= 2 ? 2 : 1;  // __launch_bounds__ minimum CTAs per SM
      }
    }
  }
  return best;
}

// In-place Stockham sub-stages s_begin..s_end-1 of DFT_L on COLS rows of the tile A[row][element]
// (pitch LP): KB butterfly rounds per thread, all of a stage's butterflies read into registers
// before the barrier, then written (one level of Eq. 2, per sub-stage; twiddles
// from the stage table).
std::string inplace_stages(int L, const int* R, int S, int COLS, int T, int s_begin = 0, int s_end = -1) {
  std::string s;
  if (s_end < 0) s_end = S;
  int Ns = 1;
  for (int i = 0; i < s_begin; ++i) Ns *= R[i];
  for (int i = s_begin; i < s_end; ++i) {
    const int Rs = R[i], NB = L / Rs, KB = (COLS * NB + T - 1) / T;
    const bool exact = (COLS * NB) % T == 0;
    std::string st = R"(  {  // sub-stage $I: radix $R, Ns $NS, $KB butterfly round(s) per thread
    cf v[$KB][$R];
#pragma unroll
    for (int kb = 0; kb < $KB; ++kb) {
      const int q = threadIdx.x + kb * T, ff = q / $NB, j = q - ff * $NB;
      if ($GUARD) {
#pragma unroll
        for (int r = 0; r < $R; ++r) v[kb][r] = A[SIDX(ff, j + r * $NB)];
      }
    }
    __syncthreads();
#pragma unroll
    for (int kb = 0; kb < $KB; ++kb) {
      const int q = threadIdx.x + kb * T, ff = q / $NB, j = q - ff * $NB;
      if ($GUARD) {
        const int m = j % $NS;
$TW        dft$R(v[kb]);
        const int o = (j / $NS) * $NSR + m;
#pragma unroll
        for (int r = 0; r < $R; ++r) A[SIDX(ff, o + r * $NS)] = v[kb][r];
      }
    }
    __syncthreads();
  }
)";
    const std::string tws = Ns > 1 ? "#pragma unroll\n        for (int r = 1; r < " + std::to_string(Rs) +
                                          "; ++r) v[kb][r] = cmulf(v[kb][r], tw[" + std::to_string(Ns - 1) +
                                          " + (r - 1) * " + std::to_string(Ns) + " + m]);\n"
                                    : "";
    s += subst(st, {{"I", std::to_string(i)},
                    {"KB", std::to_string(KB)},
                    {"NSR", std::to_string(Ns * Rs)},
                    {"NS", std::to_string(Ns)},
                    {"NB", std::to_string(NB)},
                    {"GUARD", exact ? "true" : "q < " + std::to_string(COLS * NB)},
                    {"TW", tws},
                    {"R", std::to_string(Rs)}});
    Ns *= Rs;
  }
  return s;
}

// Single-pass kernel generated for N (N <= 4096 with prime factors 11..kJitMaxPrime): FPB whole
// transforms per CTA (the jit_pass_geo geometry with the transforms as the tile's rows), the
// contiguous FPB*N tile loaded and stored with coalesced accesses, in-place sub-stages, the
// inverse's conjugation a separate entry point.
// Fused single-pass geometry: T = FPB * (N / R_0) threads, thread (f, j) = stage 0's butterfly j of
// transform f (lanes along j: its loads a[f N + j + r N/R_0] are coalesced), the last sub-stage
// stores a[f N + j + r Ns] from registers (also coalesced along j).  cols == 0: none.
PassGeo jit_single_geo_fused(int N, const int* R, int S) {
  PassGeo best;
  // a single-stage N (a prime) has one butterfly per transform: lanes would walk transforms at
  // stride N, uncoalesced (measured 2x slower for 11, 13, 61) -- the generic kernel stays there
  if (S < 2) return best;
  const int nb0 = N / R[0], lp = jit_pitch(N, R, true);
  double bscore = -1.0;
  for (int fpb = 1; fpb <= 256; fpb *= 2) {
    const int T = fpb * nb0;
    const size_t smem = S > 1 ? (size_t)fpb * lp * 8 : 0;
    if (T > 512 || T < 32 || smem > (size_t)100 * 1024) continue;
    int vals = R[0];
    double useful = (double)fpb * N, slots = (double)T * R[0];
    bool ok = true;
    for (int q = 1; q < S; ++q) {
      const int nb = fpb * (N / R[q]), kb = (nb + T - 1) / T;
      if (kb * R[q] > (R[q] > 32 ? R[q] : 32)) ok = false;
      if (kb * R[q] > vals) vals = kb * R[q];
      useful += (double)nb * R[q];
      slots += (double)kb * T * R[q];
    }
    if (!ok) continue;
    const int regs = 2 * vals + 48;
    const int ctas_reg = 65536 / (T * (regs > 64 ? regs : 64));
    const int ctas_smem = smem ? (int)((227 * 1024) / (smem + 1024)) : 32;
    int ctas = ctas_reg < ctas_smem ? ctas_reg : ctas_smem;
    if (ctas > 32) ctas = 32;
    if (ctas < 1) continue;
    const double tile = (double)fpb * N, warps = (double)ctas * ((T + 31) / 32);
    const double score = useful / slots * ((double)T / (32.0 * ((T + 31) / 32))) +
                         0.03 * (tile < 4096 ? tile / 4096 : 1.0) + 0.06 * (warps < 24 ? warps / 24 : 1.0) +
                         (ctas >= 2 ? 0.1 : 0.0);
    if (score > bscore + 1e-9) {
      bscore = score;
      best.cols = fpb;
      best.threads = T;
      best.lp = lp;
      best.minb = ctas >= 2 ? 2 : 1;
    }
  }
  return best;
}

std::string jit_source_fused(int N, const int* R, int S, const PassGeo& g) {
  const int FPB = g.cols, T = g.threads, R0 = R[0], NB0 = N / R0, RL = R[S - 1], NBL = N / RL;
  int NsL = 1;
  for (int i = 0; i < S - 1; ++i) NsL *= R[i];
  const int KBL = (FPB * NBL + T - 1) / T;
  std::string s = "// generated by libfftc (jit.cpp) for N = " + std::to_string(N) + " (fused I/O)\n" + prelude(R, S) + jit_sidx_macro(R, true);
  s += R"(template <bool C>
__device__ __forceinline__ void body(const cf* __restrict__ in, cf* __restrict__ out, const cf* __restrict__ tw,
                                     long long batch) {
  extern __shared__ cf A[];
  constexpr int N = $N, LP = $LP, FPB = $FPB, T = $T, R0 = $R0, NB0 = $NB0;
  auto cmulf = [](cf a, cf w) { return cf{fmaf(a.x, w.x, -a.y * w.y), fmaf(a.x, w.y, a.y * w.x)}; };
  const long long f0 = (long long)blockIdx.x * FPB;
  const int nf = (int)(batch - f0 < FPB ? batch - f0 : FPB);
  const cf* gi = in + f0 * N;
  cf* go = out + f0 * N;
  {  // sub-stage 0 on the loaded elements j + r NB0 of transform f
    const int f = threadIdx.x / NB0, j = threadIdx.x - f * NB0;
    cf v[R0];
#pragma unroll
    for (int r = 0; r < R0; ++r) v[r] = f < nf ? gi[f * N + j + r * NB0] : cf{0.f, 0.f};
#pragma unroll
    for (int r = 0; r < R0; ++r) if (C) v[r].y = -v[r].y;
    dft$R0(v);
)";
  if (S == 1) {
    s += R"(    if (f < nf) {
#pragma unroll
      for (int r = 0; r < R0; ++r) go[f * N + j + r * NB0] = cf{v[r].x, C ? -v[r].y : v[r].y};
    }
  }
}
)";
  } else {
    s += R"(#pragma unroll
    for (int r = 0; r < R0; ++r) A[SIDX(f, j * R0 + r)] = v[r];
  }
  __syncthreads();
)";
    s += inplace_stages(N, R, S, FPB, T, 1, S - 1);
    s += R"(#pragma unroll
  for (int kb = 0; kb < $KBL; ++kb) {  // last sub-stage straight to HBM, lanes along j
    const int q = threadIdx.x + kb * T, ff = q / $NBL, j = q - ff * $NBL;
    if ((FPB * $NBL) % T == 0 || q < FPB * $NBL) {
      cf v[$RL];
#pragma unroll
      for (int r = 0; r < $RL; ++r) v[r] = A[SIDX(ff, j + r * $NBL)];
      const int m = j % $NSL;
#pragma unroll
      for (int r = 1; r < $RL; ++r) v[r] = cmulf(v[r], tw[$NSL - 1 + (r - 1) * $NSL + m]);
      dft$RL(v);
      if (ff < nf) {
#pragma unroll
        for (int r = 0; r < $RL; ++r) go[ff * N + j + r * $NSL] = cf{v[r].x, C ? -v[r].y : v[r].y};
      }
    }
  }
}
)";
  }
  s += R"(extern "C" __global__ void __launch_bounds__($T, $MINB) fftc_jit(const cf* __restrict__ in, cf* __restrict__ out,
    const cf* __restrict__ tw, long long batch, float) { body<false>(in, out, tw, batch); }
extern "C" __global__ void __launch_bounds__($T, $MINB) fftc_jit_c(const cf* __restrict__ in, cf* __restrict__ out,
    const cf* __restrict__ tw, long long batch, float) { body<true>(in, out, tw, batch); }
)";
  return subst(s, {{"MINB", std::to_string(g.minb)},
                   {"FPB", std::to_string(FPB)},
                   {"KBL", std::to_string(KBL)},
                   {"NBL", std::to_string(NBL)},
                   {"NSL", std::to_string(NsL)},
                   {"NB0", std::to_string(NB0)},
                   {"LP", std::to_string(g.lp)},
                   {"RL", std::to_string(RL)},
                   {"R0", std::to_string(R0)},
                   {"T", std::to_string(T)},
                   {"N", std::to_string(N)}});
}

// the geometry jit_source and jit_get use: the fused kernel's when one exists (FFTC_JIT_GENERIC=1
// forces the generic one)
PassGeo jit_single_geo(int N, const int* R, int S, bool* fused) {
  *fused = false;
  if (!getenv("FFTC_JIT_GENERIC")) {
    const PassGeo gf = jit_single_geo_fused(N, R, S);
    if (gf.cols > 0) {
      *fused = true;
      return gf;
    }
  }
  return jit_pass_geo(N, R, S, 1, true);
}

std::string jit_source(int N) {
  int R[32];
  const int S = jit_radices(N, R, 32);
  if (S < 0) return "";
  return jit_source_r(N, R, S);
}

std::string jit_source_r(int N, const int* R, int S) {
  bool fused = false;
  const PassGeo g = jit_single_geo(N, R, S, &fused);
  if (g.cols <= 0) return "";
  if (fused) return jit_source_fused(N, R, S, g);
  const int FPB = g.cols, T = g.threads, EL = (FPB * N + T - 1) / T;
  const int UR = EL < kJitLoadRound ? EL : kJitLoadRound;
  std::string s = "// generated by libfftc (jit.cpp) for N = " + std::to_string(N) + "\n" + prelude(R, S) + jit_sidx_macro(R, true);
  s += R"(template <bool C>
__device__ __forceinline__ void body(const cf* __restrict__ in, cf* __restrict__ out, const cf* __restrict__ tw,
                                     long long batch) {
  extern __shared__ cf A[];
  constexpr int N = $N, LP = $LP, FPB = $FPB, T = $T, EL = $EL, UR = $UR;
  auto cmulf = [](cf a, cf w) { return cf{fmaf(a.x, w.x, -a.y * w.y), fmaf(a.x, w.y, a.y * w.x)}; };
  const long long f0 = (long long)blockIdx.x * FPB;
  const int nf = (int)(batch - f0 < FPB ? batch - f0 : FPB);
  const int lim = nf * N;  // valid elements of this tile (the last tile may be ragged)
  const cf* gi = in + f0 * N;
  cf* go = out + f0 * N;
#pragma unroll
  for (int u0 = 0; u0 < EL; u0 += UR) {
    cf v[UR];
#pragma unroll
    for (int k = 0; k < UR; ++k) {
      const int e = threadIdx.x + (u0 + k) * T;
      if (u0 + k < EL) v[k] = e < lim ? gi[e] : cf{0.f, 0.f};
    }
#pragma unroll
    for (int k = 0; k < UR; ++k) {
      const int e = threadIdx.x + (u0 + k) * T;
      if (u0 + k < EL && ((FPB * N) % T == 0 || e < FPB * N)) {
        cf x = v[k];
        if (C) x.y = -x.y;
        A[SIDX(e / N, e % N)] = x;
      }
    }
  }
  __syncthreads();
)";
  s += inplace_stages(N, R, S, FPB, T);
  s += R"(#pragma unroll
  for (int u = 0; u < EL; ++u) {
    const int e = threadIdx.x + u * T;
    if (e < lim) { const cf a = A[SIDX(e / N, e % N)]; go[e] = cf{a.x, C ? -a.y : a.y}; }
  }
}
extern "C" __global__ void __launch_bounds__($T, $MINB) fftc_jit(const cf* __restrict__ in, cf* __restrict__ out,
    const cf* __restrict__ tw, long long batch, float) { body<false>(in, out, tw, batch); }
extern "C" __global__ void __launch_bounds__($T, $MINB) fftc_jit_c(const cf* __restrict__ in, cf* __restrict__ out,
    const cf* __restrict__ tw, long long batch, float) { body<true>(in, out, tw, batch); }
)";
  return subst(s, {{"MINB", std::to_string(g.minb)},
                   {"FPB", std::to_string(FPB)},
                   {"LP", std::to_string(g.lp)},
                   {"UR", std::to_string(UR)},
                   {"EL", std::to_string(EL)},
                   {"T", std::to_string(T)},
                   {"N", std::to_string(N)}});
}

// Geometry of the fused pass kernel: T = COLS * (L / R_0) threads, so thread (f, j) holds exactly
// stage 0's butterfly j of column f when it loads rows j + r L/R_0 -- the first sub-stage runs on
// the loaded registers and the last one stores to HBM from registers (later passes), two
// shared-memory round trips and a barrier fewer than the generic kernel.  cols == 0: none.
PassGeo jit_pass_geo_fused(int L, const int* R, int S) {
  PassGeo best;
  if (S < 2) return best;
  const int nb0 = L / R[0], lp = jit_pitch(L, R, false);
  double bscore = -1.0;
  for (int cols = 2; cols <= 128; cols *= 2) {  // < 8 columns only when nothing wider fits (long passes)
    const int T = cols * nb0;
    const size_t smem = (size_t)cols * lp * 8;
    if (T > 512 || T < 64 || T % 32 || smem > (size_t)100 * 1024) continue;
    int vals = R[0];
    double useful = 0.0, slots = 0.0;
    bool ok = true;
    for (int q = 1; q < S; ++q) {
      const int nb = cols * (L / R[q]), kb = (nb + T - 1) / T;
      if (kb * R[q] > 32) ok = false;
      if (kb * R[q] > vals) vals = kb * R[q];
      useful += (double)nb * R[q];
      slots += (double)kb * T * R[q];
    }
    if (!ok) continue;
    const int regs = 2 * vals + 48;
    const int ctas_reg = 65536 / (T * (regs > 64 ? regs : 64));
    const int ctas_smem = (int)((227 * 1024) / (smem + 1024));
    const int ctas = ctas_reg < ctas_smem ? ctas_reg : ctas_smem;
    if (ctas < 1) continue;
    const double tile = (double)cols * L, warps = (double)ctas * T / 32.0;
    const double score = useful / slots + 0.03 * (tile < 4096 ? tile / 4096 : 1.0) +
                         0.06 * (warps < 24 ? warps / 24 : 1.0) + (ctas >= 2 ? 0.1 : 0.0) - (cols < 8 ? 0.5 : 0.0);
    if (score > bscore + 1e-9) {
      bscore = score;
      best.cols = cols;
      best.threads = T;
      best.lp = lp;
      best.minb = ctas >= 2 ? 2 : 1;
    }
  }
  return best;
}

// The fused pass kernel (see jit_pass_geo_fused); same entry points and arguments as the
// generic one below.
std::string jit_pass_source_fused(int L, const int* R, int S, const PassGeo& g) {
  const int COLS = g.cols, T = g.threads, R0 = R[0], NB0 = L / R0, RL = R[S - 1], NBL = L / RL;
  int NsL = 1;
  for (int i = 0; i < S - 1; ++i) NsL *= R[i];
  const int KBL = (COLS * NBL + T - 1) / T;
  std::string s = "// generated by libfftc (jit.cpp): fused pass of length " + std::to_string(L) + "\n" + prelude(R, S) + jit_sidx_macro(R, false);
  s += R"(template <bool FIRST, bool CI, bool CO>
__device__ __forceinline__ void pass_body(const cf* __restrict__ in, cf* __restrict__ out, const cf* __restrict__ tw,
    const cf* __restrict__ twA, const cf* __restrict__ twB, long long N, int Ns, int tws, int tiles, float csign_in,
    float csign_out) {
  extern __shared__ cf A[];
  constexpr int L = $L, LP = $LP, COLS = $COLS, T = $T, R0 = $R0, NB0 = $NB0;
  const int NB = (int)(N / L);  // columns of this pass (< 2^31)
  const int bt = (int)(blockIdx.x / tiles);
  const int c0 = (int)(blockIdx.x - bt * tiles) * COLS;
  const int nc = NB - c0 < COLS ? NB - c0 : COLS;
  const int f = threadIdx.x % COLS, j0 = threadIdx.x / COLS;  // column, stage-0 butterfly
  const int c = c0 + f;
  const bool fok = f < nc;
  const long long amask = (1LL << tws) - 1;
  auto root = [&](long long e) { const cf p = twA[e & amask], q = twB[e >> tws];
    return cf{fmaf(p.x, q.x, -p.y * q.y), fmaf(p.x, q.y, p.y * q.x)}; };
  auto cmulf = [](cf a, cf w) { return cf{fmaf(a.x, w.x, -a.y * w.y), fmaf(a.x, w.y, a.y * w.x)}; };
  {  // sub-stage 0 on the loaded rows j0 + r NB0 of column f
    cf v[R0];
    const cf* gp = in + (long long)bt * N + c + (long long)j0 * NB;
    const long long gstep = (long long)NB0 * NB;
#pragma unroll
    for (int r = 0; r < R0; ++r) v[r] = fok ? gp[r * gstep] : cf{0.f, 0.f};
#pragma unroll
    for (int r = 0; r < R0; ++r) if (CI) v[r].y = -v[r].y;
    if (!FIRST) {  // input twiddle w^{m (j0 + r NB0)} = w^{m j0} (w^{m NB0})^r, m = c mod Ns
      const int cm = c - (c / Ns) * Ns;
      cf st[R0];
      st[0] = root((long long)cm * j0);
      st[1] = root((long long)cm * NB0);
#pragma unroll
      for (int r = 2; r < R0; ++r) { int hb = 1; while (2 * hb <= r) hb *= 2;
        st[r] = r == hb ? cmulf(st[hb / 2], st[hb / 2]) : cmulf(st[hb], st[r - hb]); }
      v[0] = cmulf(v[0], st[0]);
#pragma unroll
      for (int r = 1; r < R0; ++r) v[r] = cmulf(v[r], cmulf(st[0], st[r]));
    }
    dft$R0(v);
#pragma unroll
    for (int r = 0; r < R0; ++r) A[SIDX(f, j0 * R0 + r)] = v[r];
  }
  __syncthreads();
)";
  s += inplace_stages(L, R, S, COLS, T, 1, S - 1);
  s += R"(  cf* go = out + (long long)bt * N;
  if (FIRST) {  // last sub-stage straight to HBM: column c's outputs are contiguous at c L + row, so
                // butterfly (column ff, j) with lanes walking j stores rows j + r NsL coalesced
#pragma unroll
    for (int kb = 0; kb < $KBL; ++kb) {
      const int q = threadIdx.x + kb * T, ff = q / $NBL, j = q - ff * $NBL;
      if ((COLS * $NBL) % T == 0 || q < COLS * $NBL) {
        cf v[$RL];
#pragma unroll
        for (int r = 0; r < $RL; ++r) v[r] = A[SIDX(ff, j + r * $NBL)];
        const int m = j % $NSL;
#pragma unroll
        for (int r = 1; r < $RL; ++r) v[r] = cmulf(v[r], tw[$NSL - 1 + (r - 1) * $NSL + m]);
        dft$RL(v);
        if (ff < nc) {
          cf* gs = go + (long long)(c0 + ff) * L + j;
#pragma unroll
          for (int r = 0; r < $RL; ++r) gs[r * $NSL] = cf{v[r].x, CO ? -v[r].y : v[r].y};
        }
      }
    }
  } else {  // last sub-stage from shared memory straight to HBM: butterfly (column ff, j), lanes walk ff
#pragma unroll
    for (int kb = 0; kb < $KBL; ++kb) {
      const int q = threadIdx.x + kb * T, ff = q % COLS, j = q / COLS;
      if ((COLS * $NBL) % T == 0 || q < COLS * $NBL) {
        cf v[$RL];
#pragma unroll
        for (int r = 0; r < $RL; ++r) v[r] = A[SIDX(ff, j + r * $NBL)];
        const int m = j % $NSL;
#pragma unroll
        for (int r = 1; r < $RL; ++r) v[r] = cmulf(v[r], tw[$NSL - 1 + (r - 1) * $NSL + m]);
        dft$RL(v);
        if (ff < nc) {  // output row j + r NsL of column cc at (cc div Ns) Ns L + (cc mod Ns) + row Ns
          const int cc = c0 + ff, cq = cc / Ns, cm = cc - cq * Ns;
          cf* gs = go + (long long)cq * Ns * L + cm + (long long)j * Ns;
#pragma unroll
          for (int r = 0; r < $RL; ++r) gs[(long long)r * $NSL * Ns] = cf{v[r].x, CO ? -v[r].y : v[r].y};
        }
      }
    }
  }
}
)";
  s += R"(#define FFTC_PASS_ARGS const cf* __restrict__ in, cf* __restrict__ out, const cf* __restrict__ tw, \
    const cf* __restrict__ twA, const cf* __restrict__ twB, long long N, int Ns, int tws, int tiles, float csign_in, \
    float csign_out
#define FFTC_PASS_ENTRY(NAME, FIRST, CI, CO) \
  extern "C" __global__ void __launch_bounds__($T, $MINB) NAME(FFTC_PASS_ARGS) { \
    pass_body<FIRST, CI, CO>(in, out, tw, twA, twB, N, Ns, tws, tiles, csign_in, csign_out); }
FFTC_PASS_ENTRY(fftc_jit_pass, false, false, false)
FFTC_PASS_ENTRY(fftc_jit_pass_co, false, false, true)
FFTC_PASS_ENTRY(fftc_jit_pass_first, true, false, false)
FFTC_PASS_ENTRY(fftc_jit_pass_first_ci, true, true, false)
FFTC_PASS_ENTRY(fftc_jit_pass_first_cico, true, true, true)
FFTC_PASS_ENTRY(fftc_jit_pass_first_co, true, false, true)
)";
  return subst(s, {{"MINB", std::to_string(g.minb)},
                   {"COLS", std::to_string(COLS)},
                   {"KBL", std::to_string(KBL)},
                   {"NBL", std::to_string(NBL)},
                   {"NSL", std::to_string(NsL)},
                   {"NB0", std::to_string(NB0)},
                   {"LP", std::to_string(g.lp)},
                   {"RL", std::to_string(RL)},
                   {"R0", std::to_string(R0)},
                   {"T", std::to_string(T)},
                   {"L", std::to_string(L)}});
}

// One pass of the runtime multi-pass path (the kernel of gpass.cu) with L, its radices and
// the tile geometry compiled in: straight-line codelets (any prime up to kJitMaxPrime), every
// loop trip count and divisor a compile-time constant.  Ns, the twiddle split and the sizes
// stay runtime arguments, so one kernel serves every pass of that length.  Pass s is one level
// of Eq. 2 at the pass level: column c reads a[c + r NB], multiplies by
// w_{Ns L}^{(c mod Ns) r}, runs DFT_L as in-place Stockham sub-stages, writes the autosort
// position (c div Ns) Ns L + (c mod Ns) + r Ns.  Each thread loads and stores ONE column f
// (rows r = rs + u RSTEP), so its twiddles are w^{m rs} times powers of w^{m RSTEP} (a tree:
// powers 2^b looked up once per thread, every other one a single product).
// (the fused variant, jit_pass_source_fused, is used whenever its geometry exists)
std::string jit_pass_source(int L, const int* R, int S) {
  if (!getenv("FFTC_JIT_PASS_GENERIC")) {
    const PassGeo gf = jit_pass_geo_fused(L, R, S);
    if (gf.cols > 0) return jit_pass_source_fused(L, R, S, gf);
  }
  const PassGeo g = jit_pass_geo(L, R, S, 8, false);
  if (g.cols <= 0) return "";
  const int COLS = g.cols, T = g.threads, RSTEP = T / COLS, E = (L + RSTEP - 1) / RSTEP;
  const int UR = E < kJitLoadRound ? E : kJitLoadRound;
  std::string s = "// generated by libfftc (jit.cpp): pass of length " + std::to_string(L) + "\n" + prelude(R, S) + jit_sidx_macro(R, false);
  // the body is a template on FIRST (pass 0: Ns = 1, no input twiddle, contiguous column
  // outputs); fftc_jit_pass_first / fftc_jit_pass instantiate it, so neither carries the other's
  // code under a runtime predicate
  s += R"(template <bool FIRST, bool CI, bool CO>
__device__ __forceinline__ void pass_body(const cf* __restrict__ in, cf* __restrict__ out, const cf* __restrict__ tw,
    const cf* __restrict__ twA, const cf* __restrict__ twB, long long N, int Ns, int tws, int tiles, float csign_in,
    float csign_out) {
  extern __shared__ cf A[];
  constexpr int L = $L, LP = $LP, COLS = $COLS, T = $T, RSTEP = $RSTEP, E = $E, UR = $UR;
  const int NB = (int)(N / L);  // columns of this pass (< 2^31)
  const int bt = (int)(blockIdx.x / tiles);
  const int c0 = (int)(blockIdx.x - bt * tiles) * COLS;
  const int nc = NB - c0 < COLS ? NB - c0 : COLS;
  const int f = threadIdx.x % COLS, rs = threadIdx.x / COLS;  // this thread's column and first row
  const int c = c0 + f, cq = c / Ns, cm = c - cq * Ns;
  const bool fok = f < nc;
  const long long amask = (1LL << tws) - 1;
  auto root = [&](long long e) { const cf p = twA[e & amask], q = twB[e >> tws];
    return cf{fmaf(p.x, q.x, -p.y * q.y), fmaf(p.x, q.y, p.y * q.x)}; };
  auto cmulf = [](cf a, cf w) { return cf{fmaf(a.x, w.x, -a.y * w.y), fmaf(a.x, w.y, a.y * w.x)}; };
  {  // column f, rows r_u = rs + u RSTEP: loaded in rounds of UR (a round's loads all in flight)
    const cf* gp = in + (long long)bt * N + c + (long long)rs * NB;
    const long long gstep = (long long)RSTEP * NB;
    // input twiddle w^{m r_u}, m = c mod Ns: looked up for u = 0 mod 8, else that times
    // st[u mod 8] = w^{m (u mod 8) RSTEP} -- one lookup, the other powers as products (a tree:
    // st[k] = st[2^b] st[k - 2^b], at most three products deep)
    cf st[8];
    if (!FIRST) {
      st[1] = root((long long)cm * RSTEP);
#pragma unroll
      for (int k = 2; k < (E < 8 ? E : 8); ++k) {
        const int hb = k >= 4 ? 4 : 2;
        st[k] = k == hb ? cmulf(st[hb / 2], st[hb / 2]) : cmulf(st[hb], st[k - hb]);
      }
    }
#pragma unroll
    for (int u0 = 0; u0 < E; u0 += UR) {
      cf v[UR];
#pragma unroll
      for (int k = 0; k < UR; ++k) {
        const int u = u0 + k;
        if (u < E && (L % RSTEP == 0 || rs + u * RSTEP < L)) v[k] = fok ? gp[u * gstep] : cf{0.f, 0.f};
      }
      cf base = cf{1.f, 0.f};
#pragma unroll
      for (int k = 0; k < UR; ++k) {
        const int u = u0 + k, r = rs + u * RSTEP;
        if (u < E && (L % RSTEP == 0 || r < L)) {
          cf x = v[k];
          if (CI) x.y = -x.y;
          if (!FIRST) {
            if ((u & 7) == 0 || k == 0) base = root((long long)cm * (rs + (u & ~7) * RSTEP));
            x = (u & 7) ? cmulf(x, cmulf(base, st[u & 7])) : cmulf(x, base);
          }
          A[SIDX(f, r)] = x;  // columns >= nc carry zeros: computed, never stored to HBM
        }
      }
    }
  }
  __syncthreads();
)";
  s += inplace_stages(L, R, S, COLS, T);
  s += R"(  cf* go = out + (long long)bt * N;
  if (FIRST) {  // first pass: column c's L outputs are contiguous at c L + r (lanes walk them)
    cf* gout = go + (long long)c0 * L;
#pragma unroll 4
    for (int e = threadIdx.x; e < COLS * L; e += T) {
      const int ff = e / L, r = e - ff * L;
      if (ff < nc) { const cf a = A[SIDX(ff, r)]; gout[e] = cf{a.x, CO ? -a.y : a.y}; }
    }
  } else if (fok) {  // autosort position (c div Ns) Ns L + (c mod Ns) + r Ns (lanes walk c)
    cf* gs = go + (long long)cq * Ns * L + cm + (long long)rs * Ns;
    const long long sstep = (long long)RSTEP * Ns;
#pragma unroll
    for (int u = 0; u < E; ++u) {
      const int r = rs + u * RSTEP;
      if (L % RSTEP == 0 || r < L) { const cf a = A[SIDX(f, r)]; gs[u * sstep] = cf{a.x, CO ? -a.y : a.y}; }
    }
  }
}
#define FFTC_PASS_ARGS const cf* __restrict__ in, cf* __restrict__ out, const cf* __restrict__ tw, \
    const cf* __restrict__ twA, const cf* __restrict__ twB, long long N, int Ns, int tws, int tiles, float csign_in, \
    float csign_out
// entry points: first pass or not x conjugated input (inverse, first pass) x conjugated output
// (inverse, last pass); the sign multiplies are compiled in, not applied at run time
#define FFTC_PASS_ENTRY(NAME, FIRST, CI, CO) \
  extern "C" __global__ void __launch_bounds__($T, $MINB) NAME(FFTC_PASS_ARGS) { \
    pass_body<FIRST, CI, CO>(in, out, tw, twA, twB, N, Ns, tws, tiles, csign_in, csign_out); }
FFTC_PASS_ENTRY(fftc_jit_pass, false, false, false)
FFTC_PASS_ENTRY(fftc_jit_pass_co, false, false, true)
FFTC_PASS_ENTRY(fftc_jit_pass_first, true, false, false)
FFTC_PASS_ENTRY(fftc_jit_pass_first_ci, true, true, false)
FFTC_PASS_ENTRY(fftc_jit_pass_first_cico, true, true, true)
FFTC_PASS_ENTRY(fftc_jit_pass_first_co, true, false, true)
)";
  return subst(s, {{"MINB", std::to_string(g.minb)},
                   {"COLS", std::to_string(COLS)},
                   {"RSTEP", std::to_string(RSTEP)},
                   {"LP", std::to_string(g.lp)},
                   {"UR", std::to_string(UR)},
                   {"T", std::to_string(T)},
                   {"L", std::to_string(L)},
                   {"E", std::to_string(E)}});
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
                             int fpb, cudaError_t* err, const char* const* more = nullptr, int nmore = 0,
                             int threads = kJitThreads) {
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
  k->threads = threads;
  bool ok = setattr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)k->smem) == CUDA_SUCCESS;
  for (int i = 0; i < nmore && i < JitKernel::kVariants && ok; ++i)
    ok = getfn(&k->variant[i], mod, more[i]) == CUDA_SUCCESS &&
         setattr(k->variant[i], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)k->smem) == CUDA_SUCCESS;
  if (!ok) {
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
  int R[32];
  const int S = jit_radices(N, R, 32);
  if (S <= 0) {
    *err = cudaErrorNotSupported;
    return nullptr;
  }
  return jit_get_r(N, R, S, err);
}

const JitKernel* jit_get_r(int N, const int* R, int S, cudaError_t* err) {
  bool fused = false;
  const PassGeo g = S > 0 ? jit_single_geo(N, R, S, &fused) : PassGeo{};
  if (g.cols <= 0) {
    *err = cudaErrorNotSupported;
    return nullptr;
  }
  static const char* const names[1] = {"fftc_jit_c"};  // variant[0]: the inverse (conjugated)
  const size_t smem = (fused && S == 1) ? 0 : (size_t)g.cols * g.lp * 8;
  std::string key = std::string(fused ? "n:" : "ng:") + std::to_string(N);
  for (int i = 0; i < S; ++i) key += ":" + std::to_string(R[i]);
  return load_kernel(key, jit_source_r(N, R, S), "fftc_jit", smem, N, g.cols, err, names, 1, g.threads);
}

const JitKernel* jit_pass_get(int L, const int* R, int S, cudaError_t* err) {
  std::string key = std::string(getenv("FFTC_JIT_PASS_GENERIC") ? "pg:" : "p:") + std::to_string(L);
  for (int i = 0; i < S; ++i) key += ":" + std::to_string(R[i]);
  PassGeo g = getenv("FFTC_JIT_PASS_GENERIC") ? PassGeo{} : jit_pass_geo_fused(L, R, S);
  if (g.cols <= 0) g = jit_pass_geo(L, R, S, 8, false);
  if (g.cols <= 0) {
    *err = cudaErrorNotSupported;
    return nullptr;
  }
  // variant[first * 4 + ci * 2 + co], the combinations a plan uses (the first pass never has
  // co without being the last, but all six entry points exist)
  static const char* const names[JitKernel::kVariants] = {
      "fftc_jit_pass", "fftc_jit_pass_co", "fftc_jit_pass", "fftc_jit_pass_co",
      "fftc_jit_pass_first", "fftc_jit_pass_first_co", "fftc_jit_pass_first_ci", "fftc_jit_pass_first_cico"};
  return load_kernel(key, jit_pass_source(L, R, S), "fftc_jit_pass", (size_t)g.cols * g.lp * 8, L, g.cols, err,
                     names, JitKernel::kVariants, g.threads);
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
  // Ns = 1 only for the first pass; conj_in is set only there (the inverse's input conjugation)
  CUfunction fn = k->variant[(Ns == 1 ? 4 : 0) + (conj_in ? 2 : 0) + (conj_out ? 1 : 0)];
  const CUresult r = launch(fn, (unsigned)grid, 1, 1, (unsigned)k->threads, 1, 1, (unsigned)k->smem, (CUstream)st,
                            args, nullptr);
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
  const CUresult r = launch(conj ? k->variant[0] : k->fn, (unsigned)grid, 1, 1, (unsigned)k->threads, 1, 1,
                            (unsigned)k->smem, (CUstream)st, args, nullptr);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

const char* jit_last_log() { return g_log.c_str(); }

}  // namespace fftc
