// planner.cpp -- radix planner (host only, product path).
//
// Factors N = M K recursively (Eq. 2 "with N = MK"; the paper's
// own generator picks the split, and names the missing FFTW-style planner
// as future work).  Policy: the compiled fast
// schedule for N if there is one; otherwise a generic schedule from the codelet
// set {16, 8, 4, 2, 9, 3, 25, 5, 7} -- fewest stages, larger radices first,
// power-of-two radices before odd ones; prime factors > 7 are rejected.
// Above the single-pass limit: powers of two run the multi-pass TMA path
// (passes.cu) when it is the faster one, else the four-step with the split
// N = M K chosen below.
#include "planner.h"

#include <stdlib.h>

#include "fourstep.h"
#include "registry.h"

namespace fftc {

bool seven_smooth(int64_t n) {
  if (n < 1) return false;
  for (int p : {2, 3, 5, 7})
    while (n % p == 0) n /= p;
  return n == 1;
}

int generic_radices(int64_t N, int* R, int max) {
  if (N < 1 || !seven_smooth(N)) return -1;
  int S = 0;
  int64_t n = N;
  auto push = [&](int r) {
    if (S < max) R[S] = r;
    ++S;
    n /= r;
  };
  int a = 0;
  while (n % 2 == 0) {
    n /= 2;
    ++a;
  }
  n = N;  // recompute via pushes below
  // powers of two: 16s, then one 8/4/2 for the remainder
  int a16 = a / 4, arem = a % 4;
  for (int i = 0; i < a16; ++i) push(16);
  if (arem == 3) push(8);
  else if (arem == 2) push(4);
  else if (arem == 1) push(2);
  while (n % 9 == 0) push(9);
  if (n % 3 == 0) push(3);
  while (n % 25 == 0) push(25);
  if (n % 5 == 0) push(5);
  while (n % 7 == 0) push(7);
  return S;
}

int single_pass_radices(int64_t N, int* R, int max) {
  if (N == 1) return 0;
  if (N < 1 || !seven_smooth(N)) return -1;
  if (N <= kGenericMaxN) {
    if (const FusedEntry* e = find_fused((int)N)) {
      for (int s = 0; s < e->S && s < max; ++s) R[s] = e->R[s];
      return e->S;
    }
  }
  return generic_radices(N, R, max);
}

int top_split(int64_t N, int64_t* M, int64_t* K) {
  if (N < 1 || !seven_smooth(N)) return -1;
  if (N <= kGenericMaxN) {
    *M = N;
    *K = 1;
    return 1;
  }
  int64_t bestM = 0, bestK = 0;
  const char* force = getenv("FFTC_SPLIT_M");  // tuning: pin the top-level split
  // measured on B200 (tools/tune4.py): the strided column pass is the slower one, so keep
  // its length M near 512 (C = 8..16 columns per CTA fit in shared memory) and give the
  // row pass the rest (K <= 4096)
  auto score = [](int64_t m) { return m > 512 ? m / 512 : 512 / m; };
  for (int i = 0; i < col_count(); ++i) {
    const ColEntry* c = col_at(i);
    if (N % c->M) continue;
    if (force && atoll(force) != c->M) continue;
    const int64_t k = N / c->M;
    if (k > 0x7fffffff || !find_row((int)k)) continue;
    if (bestM == 0 || score(c->M) < score(bestM)) {
      bestM = c->M;
      bestK = k;
    }
  }
  if (bestM == 0) return -1;
  *M = bestM;
  *K = bestK;
  return 2;
}

}  // namespace fftc
