// expr.h -- FFTc factorization expressions -> radix schedule (product path, host only).
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace fftc {

// Parse an FFTc expression (Listing 1 syntax) and match it to Eq. 2 applied
// recursively.  Writes N and the radices R_0..R_{S-1} (innermost first); returns S
// (0 for a bare DFT(N): the planner chooses), or -1 with a message in err.
int expr_radices(const char* text, int64_t* N, int64_t* radices, int max, char* err, size_t errlen);

}  // namespace fftc
