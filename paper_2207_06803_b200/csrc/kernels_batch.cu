// kernels_batch.cu -- registry over the compiled single-pass schedules (product path).
#include <stdlib.h>
#include <string.h>

#include "registry.h"

namespace fftc {

extern const FusedEntry kTable_packed[], kTable_small[], kTable_mid[], kTable_large[], kTable_mixed[],
    kTable_packed_cand[];
extern const int kCount_packed, kCount_small, kCount_mid, kCount_large, kCount_mixed, kCount_packed_cand;

namespace {
struct Span {
  const FusedEntry* t;
  const int* n;
};
// kTable_packed first: its rows are the defaults for their sizes (the first row per N wins)
const Span kSpans[] = {{kTable_packed, &kCount_packed}, {kTable_small, &kCount_small}, {kTable_mid, &kCount_mid},
                       {kTable_large, &kCount_large}, {kTable_mixed, &kCount_mixed},
                       {kTable_packed_cand, &kCount_packed_cand}};
}  // namespace

int fused_count() {
  int n = 0;
  for (const auto& s : kSpans) n += *s.n;
  return n;
}

const FusedEntry* fused_at(int i) {
  if (i < 0) return nullptr;
  for (const auto& s : kSpans) {
    if (i < *s.n) return &s.t[i];
    i -= *s.n;
  }
  return nullptr;
}

const FusedEntry* find_fused(int N) {
  const int n = fused_count();
  // FFTC_KERNEL=<entry name>: pin the planner to one candidate (tuning / tests)
  if (const char* want = getenv("FFTC_KERNEL"))
    for (int i = 0; i < n; ++i)
      if (fused_at(i)->N == N && strcmp(fused_at(i)->name, want) == 0) return fused_at(i);
  for (int i = 0; i < n; ++i)
    if (fused_at(i)->N == N) return fused_at(i);
  return nullptr;
}

}  // namespace fftc
