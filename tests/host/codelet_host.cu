// Host-compiled check of the register codelets (codelets.cuh is __host__ __device__).
// Prints, for each radix, y = DFT_R(x) for x[n] = (sin(n+1), cos(2n+1)) as "R k re im" lines;
// tests/test_codelets_host.py compares them with the oracle.
#include <cmath>
#include <cstdio>
#include "../../paper_2207_06803_b200/csrc/codelets.cuh"
using namespace fftc;
template <int R> void run() {
  float2 v[R];
  for (int n = 0; n < R; ++n) v[n] = make_float2(std::sin(n + 1.0f), std::cos(2.0f * n + 1.0f));
  Codelet<R>::run(v);
  for (int k = 0; k < R; ++k) printf("%d %d %.9e %.9e\n", R, k, v[k].x, v[k].y);
}
int main() {
  run<2>(); run<3>(); run<4>(); run<5>(); run<6>(); run<7>(); run<8>(); run<9>(); run<10>();
  run<12>(); run<14>(); run<15>(); run<16>(); run<20>(); run<25>(); run<27>(); run<32>();
  return 0;
}
