/*
 * oracle/oracle.c -- CPU oracle for the batched 1D complex DFT (TEST INFRASTRUCTURE ONLY).
 *
 * This file is test infrastructure.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call it.  The
 * product path (libfftc.so, paper_2207_06803_b200/) never links, imports or
 * executes anything under oracle/, and this file shares no code, header,
 * table or constant generator with it.
 *
 * Everything is double precision, computed with -O2 -ffp-contract=off so the
 * result is bit-reproducible on one host.  Inputs are the fp32 interleaved
 * (re, im) arrays the GPU receives, upcast exactly to double.
 *
 * Paper: /root/reference/PAPER.md (arXiv 2207.06803, FFTc).
 *   P:42-47  (§Background)   DFT_N[m,n] = w_N^{mn}, w_N = exp(-2*pi*i/N);
 *                             "a direct computation ... is the multiplication
 *                             a DFT matrix by the input vector x".
 *   P:70-76  (§Background, Eq. 2)
 *                             DFT_N = (DFT_K (x) I_M) D^N_M (I_K (x) DFT_M) Pi^N_K,
 *                             N = MK, general-radix decimation in time, applied
 *                             recursively.
 * Readings: sign=-1 is the paper's forward transform, sign=+1
 * the unnormalised inverse exp(+2*pi*i/N); D^N_M holds w_N^{b*j} at diagonal
 * position b*M+j; Pi^N_K gathers (Pi x)[r*M+q] = x[q*K+r].
 *
 * Pins (tests/test_oracle.py): Eq. 1's printed factors and product, Listing 1
 * input, closed forms (delta, constant, tone, zero), Parseval, linearity,
 * Hermitian symmetry, shift theorem, round trip, O2 == O1, O1 == numpy.fft.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { double re, im; } cplx;

static cplx cmul(cplx a, cplx b) {
  cplx r;
  r.re = a.re * b.re - a.im * b.im;
  r.im = a.re * b.im + a.im * b.re;
  return r;
}

/* w_N^e for e in [0, N): per-entry cos/sin of the reduced angle 2*pi*e/N
 * (no recurrence, so no phase drift).  w = exp(sign * 2*pi*i/N). */
static cplx* root_table(int64_t N, int sign) {
  cplx* w = (cplx*)malloc(sizeof(cplx) * (size_t)N);
  if (!w) return NULL;
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t e = 0; e < N; ++e) {
    double a = two_pi * (double)e / (double)N;
    w[e].re = cos(a);
    w[e].im = (double)sign * sin(a);
  }
  return w;
}

/* ---------------------------------------------------------------- O1 ----
 * Naive O(N^2) DFT, the definition written out:
 *   Y[k] = sum_{n=0}^{N-1} X[n] * w_N^{(n*k) mod N},  accumulated in index order.
 * x: fp32 interleaved [batch][N]; y: double interleaved [nidx][N];
 * idx: which transforms (NULL -> all, nidx ignored and taken as batch).     */
void oracle_dft_naive(const float* x, double* y, int64_t N, int64_t batch, int sign,
                      const int64_t* idx, int64_t nidx) {
  if (N <= 0) return;
  int64_t nt = idx ? nidx : batch;
  cplx* w = root_table(N, sign);
  #pragma omp parallel for schedule(dynamic)
  for (int64_t t = 0; t < nt; ++t) {
    int64_t b = idx ? idx[t] : t;
    const float* xb = x + 2 * b * N;
    double* yb = y + 2 * t * N;
    for (int64_t k = 0; k < N; ++k) {
      cplx acc = {0.0, 0.0};
      for (int64_t n = 0; n < N; ++n) {
        cplx xn = {(double)xb[2 * n], (double)xb[2 * n + 1]};
        int64_t e = (int64_t)(((unsigned __int128)n * (unsigned __int128)k) % (unsigned __int128)N);
        cplx p = cmul(xn, w[e]);
        acc.re += p.re;
        acc.im += p.im;
      }
      yb[2 * k] = acc.re;
      yb[2 * k + 1] = acc.im;
    }
  }
  free(w);
}

/* One output bin of one transform by direct O(N) summation, twiddle angle
 * taken per term from the int64-reduced exponent (n*k) mod N (definition,
 * P:44-46).  Used where N is too large for a table (N = 2^30). */
void oracle_spot_bin(const float* x, int64_t N, int64_t k, int sign, double* re, double* im) {
  const double two_pi = 6.283185307179586476925286766559;
  double sr = 0.0, si = 0.0;
  #pragma omp parallel for reduction(+ : sr, si) schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    int64_t e = (int64_t)(((unsigned __int128)n * (unsigned __int128)k) % (unsigned __int128)N);
    double a = two_pi * (double)e / (double)N;
    cplx wv = {cos(a), (double)sign * sin(a)};
    cplx xn = {(double)x[2 * n], (double)x[2 * n + 1]};
    cplx p = cmul(xn, wv);
    sr += p.re;
    si += p.im;
  }
  *re = sr;
  *im = si;
}

/* ---------------------------------------------------------------- O2 ----
 * Recursive Cooley-Tukey, Eq. 2 read literally, with K the
 * smallest prime factor of N and M = N/K:
 *   Pi^N_K then I_K (x) DFT_M : y_r = DFT_M([x[r], x[r+K], ..., x[r+(M-1)K]])
 *   D^N_M                      : y_r[j] *= w_N^{(r*j) mod N}   (position r*M+j)
 *   DFT_K (x) I_M              : X[j + M*k1] = sum_r y_r[j] * w_N^{(r*k1*M) mod N}
 * Prime N is the base case and uses the naive sum (O1's formula).
 * w_N^e is read from the top-level table: w_{N'}^e = w_{Ntop}^{e*ws}.
 * in: stride xs; out: contiguous N; scratch: >= 2N.                        */
static int64_t smallest_prime_factor(int64_t n) {
  if (n % 2 == 0) return 2;
  for (int64_t p = 3; p * p <= n; p += 2)
    if (n % p == 0) return p;
  return n;
}

static void ct_rec(const cplx* x, int64_t xs, cplx* out, int64_t N, const cplx* w, int64_t ws,
                   cplx* scratch) {
  if (N == 1) {
    out[0] = x[0];
    return;
  }
  int64_t K = smallest_prime_factor(N);
  int64_t M = N / K;
  if (K == N) { /* prime: naive DFT_N */
    for (int64_t k = 0; k < N; ++k) {
      cplx acc = {0.0, 0.0};
      for (int64_t n = 0; n < N; ++n) {
        cplx p = cmul(x[n * xs], w[((n * k) % N) * ws]);
        acc.re += p.re;
        acc.im += p.im;
      }
      out[k] = acc;
    }
    return;
  }
  cplx* y = scratch; /* y[r*M + j], r < K, j < M */
  for (int64_t r = 0; r < K; ++r)
    ct_rec(x + r * xs, xs * K, y + r * M, M, w, ws * K, scratch + N);
  for (int64_t r = 1; r < K; ++r)
    for (int64_t j = 1; j < M; ++j)
      y[r * M + j] = cmul(y[r * M + j], w[((r * j) % N) * ws]);
  for (int64_t k1 = 0; k1 < K; ++k1)
    for (int64_t j = 0; j < M; ++j) {
      cplx acc = {0.0, 0.0};
      for (int64_t r = 0; r < K; ++r) {
        cplx p = cmul(y[r * M + j], w[((r * k1 * M) % N) * ws]);
        acc.re += p.re;
        acc.im += p.im;
      }
      out[j + M * k1] = acc;
    }
}

/* Batched O2.  x: fp32 interleaved [batch][N]; y: double interleaved
 * [batch][N].  nthreads <= 0 -> OpenMP default.  Returns 0, or -1 on OOM. */
int oracle_fft_ct(const float* x, double* y, int64_t N, int64_t batch, int sign, int nthreads) {
  if (N <= 0 || batch <= 0) return 0;
  cplx* w = root_table(N, sign);
  if (!w) return -1;
  int fail = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  #pragma omp parallel
  {
    cplx* xin = (cplx*)malloc(sizeof(cplx) * (size_t)N);
    cplx* scratch = (cplx*)malloc(sizeof(cplx) * (size_t)(2 * N + 2));
    if (!xin || !scratch) {
      #pragma omp atomic write
      fail = 1;
    } else {
      #pragma omp for schedule(dynamic)
      for (int64_t b = 0; b < batch; ++b) {
        const float* xb = x + 2 * b * N;
        for (int64_t n = 0; n < N; ++n) {
          xin[n].re = (double)xb[2 * n];
          xin[n].im = (double)xb[2 * n + 1];
        }
        ct_rec(xin, 1, (cplx*)(y + 2 * b * N), N, w, 1, scratch);
      }
    }
    free(xin);
    free(scratch);
  }
  free(w);
  return fail ? -1 : 0;
}

/* Same as oracle_fft_ct but on a double interleaved input (used to apply the
 * inverse to a double result, e.g. round trips inside the oracle's own pins). */
int oracle_fft_ct_f64(const double* x, double* y, int64_t N, int64_t batch, int sign,
                      int nthreads) {
  if (N <= 0 || batch <= 0) return 0;
  cplx* w = root_table(N, sign);
  if (!w) return -1;
  int fail = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  #pragma omp parallel
  {
    cplx* scratch = (cplx*)malloc(sizeof(cplx) * (size_t)(2 * N + 2));
    if (!scratch) {
      #pragma omp atomic write
      fail = 1;
    } else {
      #pragma omp for schedule(dynamic)
      for (int64_t b = 0; b < batch; ++b)
        ct_rec((const cplx*)(x + 2 * b * N), 1, (cplx*)(y + 2 * b * N), N, w, 1, scratch);
    }
    free(scratch);
  }
  free(w);
  return fail ? -1 : 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
