// codelets.cuh -- register-resident DFT_R codelets for sm_100a (product path).
//
// A codelet computes y = DFT_R x in registers, natural order in and out, in the
// forward direction w_R = exp(-2*pi*i/R).  The inverse is
// obtained by the executor as conj(DFT(conj(x))), so only forward codelets exist.
//
// Composite R is built at compile time by the paper's Eq. 2 applied
// inside the register file:  DFT_R = (DFT_K (x) I_M) D^R_M (I_K (x) DFT_M) Pi^R_K
// with R = M K: gather at stride K (Pi), M-point codelets on each of the K
// sub-vectors (I_K (x) DFT_M), twiddles w_R^{r j} at position r M + j (D^R_M),
// K-point codelets across them (DFT_K (x) I_M).  Trivial twiddles (w^0, +-1,
// +-i, the eighth roots) are resolved at compile time.  Odd primes use the
// conjugate-pair symmetric form of the DFT definition.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>
#include <utility>

#ifndef FFTC_HD
#define FFTC_HD __host__ __device__ __forceinline__
#endif

namespace fftc {

// ---------------------------------------------------------------- compile-time helpers
template <int N, int I = 0, class F>
FFTC_HD void sfor(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    sfor<N, I + 1>(f);
  }
}

constexpr double kPi = 3.14159265358979323846264338327950288;

// Taylor series on [-pi, pi]; 40 terms are far below double rounding there.
constexpr double taylor_sin(double x) {
  double term = x, sum = x;
  for (int n = 1; n < 40; ++n) {
    term *= -x * x / double((2 * n) * (2 * n + 1));
    sum += term;
  }
  return sum;
}
constexpr double taylor_cos(double x) {
  double term = 1.0, sum = 1.0;
  for (int n = 1; n < 40; ++n) {
    term *= -x * x / double((2 * n - 1) * (2 * n));
    sum += term;
  }
  return sum;
}
// cos / sin of 2*pi*e/R with the exponent reduced mod R first (exact integer reduction).
constexpr double cos2pi(long long e, long long R) {
  e %= R;
  if (e < 0) e += R;
  double t = double(e) / double(R);
  if (t > 0.5) t -= 1.0;
  return taylor_cos(2.0 * kPi * t);
}
constexpr double sin2pi(long long e, long long R) {
  e %= R;
  if (e < 0) e += R;
  double t = double(e) / double(R);
  if (t > 0.5) t -= 1.0;
  return taylor_sin(2.0 * kPi * t);
}

constexpr int smallest_factor(int n) {
  for (int p = 2; p * p <= n; ++p)
    if (n % p == 0) return p;
  return n;
}
constexpr bool is_prime(int n) { return n >= 2 && smallest_factor(n) == n; }
// Outer factor K of a composite codelet R = M*K: prefer 4, then 2, then the smallest prime.
constexpr int codelet_outer(int R) {
  if (R % 4 == 0 && R > 4) return 4;
  return smallest_factor(R);
}

// ---------------------------------------------------------------- complex helpers
// FFTC_PACKED: on the device, complex arithmetic uses sm_100's paired FP32 instructions
// (add/sub/mul/fma.rn.f32x2 -> FADD2 / FMUL2 / FFMA2 on a (re, im) register pair; ptxas folds
// the component swaps and negations of +-i products and the re/im broadcasts of a complex
// multiply into operand modifiers), about half the FP32 instructions of the scalar form.  Each
// lane op is the same IEEE round-to-nearest operation as the scalar one; only FMA contraction
// differs.  The host build (codelet tests) always takes the scalar form.
#ifndef FFTC_PACKED
#define FFTC_PACKED 0  // per translation unit: kernels_packed.cu sets 1 (faster only where issue-bound)
#endif
#if defined(__CUDA_ARCH__) && FFTC_PACKED
#define FFTC_PK 1
typedef unsigned long long fftc_u64;
__device__ __forceinline__ fftc_u64 pk2(float a, float b) {
  fftc_u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(fftc_u64 r) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
  return make_float2(a, b);
}
__device__ __forceinline__ fftc_u64 add2(fftc_u64 a, fftc_u64 b) {
  fftc_u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ fftc_u64 sub2(fftc_u64 a, fftc_u64 b) {
  fftc_u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ fftc_u64 mul2(fftc_u64 a, fftc_u64 b) {
  fftc_u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ fftc_u64 fma2(fftc_u64 a, fftc_u64 b, fftc_u64 c) {
  fftc_u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
#else
#define FFTC_PK 0
#endif

FFTC_HD float2 cadd(float2 a, float2 b) {
#if FFTC_PK
  return upk2(add2(pk2(a.x, a.y), pk2(b.x, b.y)));
#else
  return make_float2(a.x + b.x, a.y + b.y);
#endif
}
FFTC_HD float2 csub(float2 a, float2 b) {
#if FFTC_PK
  return upk2(sub2(pk2(a.x, a.y), pk2(b.x, b.y)));
#else
  return make_float2(a.x - b.x, a.y - b.y);
#endif
}
// a * b = a.x (b.x, b.y) + a.y (-b.y, b.x)
FFTC_HD float2 cmul(float2 a, float2 b) {
#if FFTC_PK
  return upk2(fma2(pk2(a.y, a.y), pk2(-b.y, b.x), mul2(pk2(a.x, a.x), pk2(b.x, b.y))));
#else
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
#endif
}
// acc + c * x for a real scalar c
FFTC_HD float2 cfma_r(float c, float2 x, float2 acc) {
#if FFTC_PK
  return upk2(fma2(pk2(c, c), pk2(x.x, x.y), pk2(acc.x, acc.y)));
#else
  return make_float2(fmaf(c, x.x, acc.x), fmaf(c, x.y, acc.y));
#endif
}
FFTC_HD float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
FFTC_HD float2 cscale(float2 a, float s) {
#if FFTC_PK
  return upk2(mul2(pk2(a.x, a.y), pk2(s, s)));
#else
  return make_float2(a.x * s, a.y * s);
#endif
}
// -i * a
FFTC_HD float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }
// +i * a
FFTC_HD float2 mul_pi(float2 a) { return make_float2(-a.y, a.x); }

// a * w_R^E, forward root w_R = exp(-2 pi i / R), E and R compile-time.
template <int E, int R>
FFTC_HD float2 mul_root(float2 a) {
  constexpr int e = ((E % R) + R) % R;
  if constexpr (e == 0) {
    return a;
  } else if constexpr ((8 * e) % R == 0) {
    constexpr int k8 = (8 * e) / R;  // angle = -k8 * pi / 4
    constexpr float h = 0.70710678118654752440f;
    if constexpr (k8 == 2) return mul_mi(a);
    else if constexpr (k8 == 4) return make_float2(-a.x, -a.y);
    else if constexpr (k8 == 6) return mul_pi(a);
    else if constexpr (k8 == 1) return cscale(cadd(a, mul_mi(a)), h);  // ((x + y) h, (y - x) h)
    else if constexpr (k8 == 3) return cscale(csub(mul_mi(a), a), h);   // ((y - x) h, -(x + y) h)
    else if constexpr (k8 == 5) return cscale(csub(mul_pi(a), a), h);   // (-(x + y) h, (x - y) h)
    else return cscale(cadd(a, mul_pi(a)), h);                          // k8 == 7: ((x - y) h, (x + y) h)
  } else {
    constexpr float c = float(cos2pi(e, R));
    constexpr float s = float(-sin2pi(e, R));
#if FFTC_PK
    return upk2(fma2(pk2(a.x, a.x), pk2(c, s), mul2(pk2(a.y, a.y), pk2(-s, c))));
#else
    return make_float2(fmaf(a.x, c, -a.y * s), fmaf(a.x, s, a.y * c));
#endif
  }
}

// ---------------------------------------------------------------- codelets
template <int R, class Enable = void>
struct Codelet;

template <>
struct Codelet<1> {
  FFTC_HD static void run(float2*) {}
};

template <>
struct Codelet<2> {
  FFTC_HD static void run(float2* v) {
    float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <>
struct Codelet<4> {
  FFTC_HD static void run(float2* v) {
    float2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    float2 t2 = cadd(v[1], v[3]), t3 = csub(v[1], v[3]);
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, mul_mi(t3));
    v[3] = csub(t1, mul_mi(t3));
  }
};

// p = 3, the same symmetric form with its single sine term folded into the outputs:
//   s = x1 + x2, d = x1 - x2, y0 = x0 + s, a = x0 - s/2,
//   y1 = a - i sin(2 pi/3) d,  y2 = a + i sin(2 pi/3) d        (forward)
// each output component one FMA of the constant with a component of d (12 FP instructions
// instead of 14: the product sin(2 pi/3) d is never formed on its own).
template <>
struct Codelet<3> {
  FFTC_HD static void run(float2* v) {
    constexpr float c = float(cos2pi(1, 3));  // -1/2
    constexpr float sn = float(sin2pi(1, 3));
    const float2 sp = cadd(v[1], v[2]);
    const float2 d = csub(v[1], v[2]);
    const float2 y0 = cadd(v[0], sp);
    const float2 a = cfma_r(c, sp, v[0]);
#if FFTC_PK
    v[1] = upk2(fma2(pk2(sn, -sn), pk2(d.y, d.x), pk2(a.x, a.y)));
    v[2] = upk2(fma2(pk2(-sn, sn), pk2(d.y, d.x), pk2(a.x, a.y)));
#else
    v[1] = make_float2(fmaf(sn, d.y, a.x), fmaf(-sn, d.x, a.y));
    v[2] = make_float2(fmaf(-sn, d.y, a.x), fmaf(sn, d.x, a.y));
#endif
    v[0] = y0;
  }
};

// Odd prime p: symmetric form of the definition y_k = sum_n x_n w_p^{nk}.
//   A_k = x0 + sum_{n=1}^{h} cos(2 pi n k / p) (x_n + x_{p-n})
//   B_k =      sum_{n=1}^{h} sin(2 pi n k / p) (x_n - x_{p-n})
//   y_k = A_k - i B_k,  y_{p-k} = A_k + i B_k        (h = (p-1)/2, forward)
template <int P>
struct Codelet<P, std::enable_if_t<(P > 3) && is_prime(P)>> {
  FFTC_HD static void run(float2* v) {
    constexpr int h = (P - 1) / 2;
    float2 sp[h + 1], sm[h + 1];
    sfor<h>([&](auto n_) {
      constexpr int n = decltype(n_)::value + 1;
      sp[n] = cadd(v[n], v[P - n]);
      sm[n] = csub(v[n], v[P - n]);
    });
    float2 y0 = v[0];
    sfor<h>([&](auto n_) {
      constexpr int n = decltype(n_)::value + 1;
      y0 = cadd(y0, sp[n]);
    });
    float2 out[P];
    out[0] = y0;
    sfor<h>([&](auto k_) {
      constexpr int k = decltype(k_)::value + 1;
      float2 A = v[0], B = make_float2(0.f, 0.f);
      sfor<h>([&](auto n_) {
        constexpr int n = decltype(n_)::value + 1;
        constexpr float c = float(cos2pi((long long)n * k, P));
        constexpr float s = float(sin2pi((long long)n * k, P));
        A = cfma_r(c, sp[n], A);
        B = cfma_r(s, sm[n], B);
      });
      out[k] = cadd(A, mul_mi(B));
      out[P - k] = csub(A, mul_mi(B));
    });
    sfor<P>([&](auto k_) {
      constexpr int k = decltype(k_)::value;
      v[k] = out[k];
    });
  }
};

constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
// a^-1 mod m for gcd(a, m) == 1 (brute force: m is a codelet factor).
constexpr int inv_mod(int a, int m) {
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return m == 1 ? 0 : -1;
}

// Composite R = M*K: Eq. 2 in registers.  When gcd(K, M) = 1 the twiddle D^R_M is
// folded into index maps instead (Good-Thomas prime-factor form of the same DFT, DESIGN
// reading 19): input n = (n1 M + n2 K) mod R, output k = CRT(k mod K, k mod M), so
// w_R^{nk} = w_K^{n1 k1} w_M^{n2 k2} and no internal twiddle multiplies remain.
template <int R>
struct Codelet<R, std::enable_if_t<(R > 4) && !is_prime(R)>> {
  static constexpr int K = codelet_outer(R);
  static constexpr int M = R / K;
  static constexpr bool kPfa = gcd_c(K, M) == 1;
  FFTC_HD static void run(float2* v) {
    if constexpr (kPfa) run_pfa(v);
    else run_ct(v);
  }
  FFTC_HD static void run_pfa(float2* v) {
    constexpr int eK = M * inv_mod(M % K, K);  // = 1 mod K, 0 mod M
    constexpr int eM = K * inv_mod(K % M, M);  // = 0 mod K, 1 mod M
    float2 u[K][M];
    sfor<K>([&](auto a_) {
      constexpr int n1 = decltype(a_)::value;
      sfor<M>([&](auto b_) {
        constexpr int n2 = decltype(b_)::value;
        u[n1][n2] = v[(n1 * M + n2 * K) % R];
      });
      Codelet<M>::run(u[n1]);
    });
    sfor<M>([&](auto b_) {
      constexpr int k2 = decltype(b_)::value;
      float2 w[K];
      sfor<K>([&](auto a_) {
        constexpr int n1 = decltype(a_)::value;
        w[n1] = u[n1][k2];
      });
      Codelet<K>::run(w);
      sfor<K>([&](auto a_) {
        constexpr int k1 = decltype(a_)::value;
        v[(k1 * eK + k2 * eM) % R] = w[k1];
      });
    });
  }
  FFTC_HD static void run_ct(float2* v) {
    float2 u[K][M];
    // Pi^R_K then I_K (x) DFT_M:  u_r[q] = x[q K + r]
    sfor<K>([&](auto r_) {
      constexpr int r = decltype(r_)::value;
      sfor<M>([&](auto q_) {
        constexpr int q = decltype(q_)::value;
        u[r][q] = v[q * K + r];
      });
      Codelet<M>::run(u[r]);
    });
    // D^R_M: u_r[j] *= w_R^{r j}
    sfor<K>([&](auto r_) {
      constexpr int r = decltype(r_)::value;
      sfor<M>([&](auto j_) {
        constexpr int j = decltype(j_)::value;
        u[r][j] = mul_root<r * j, R>(u[r][j]);
      });
    });
    // DFT_K (x) I_M:  X[j + M k1] = sum_r u_r[j] w_K^{r k1}
    sfor<M>([&](auto j_) {
      constexpr int j = decltype(j_)::value;
      float2 w[K];
      sfor<K>([&](auto r_) {
        constexpr int r = decltype(r_)::value;
        w[r] = u[r][j];
      });
      Codelet<K>::run(w);
      sfor<K>([&](auto k_) {
        constexpr int k1 = decltype(k_)::value;
        v[j + M * k1] = w[k1];
      });
    });
  }
};

}  // namespace fftc
