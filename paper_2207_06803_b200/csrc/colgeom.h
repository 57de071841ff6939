// colgeom.h -- geometry of a strided column DFT launch (see colfft.cuh) (product path).
#pragma once

namespace fftc {

struct ColGeom {
  int tiles;         // column tiles (of C) per group
  long long in_g;    // input offset between groups
  long long in_s;    // input stride along the transform
  long long out_g;   // output offset between groups
  long long out_c;   // output stride between columns
  long long out_s;   // output stride along the transform (within a chunk)
  long long out_cs;  // output offset between chunks of (omask+1) outputs
  int ocl;           // log2 of the output chunk length (>= 30: no chunking)
  int tw;            // apply the twiddle
  int tw_shift;      // twiddle column index = (ci >> tw_shift) + tw_off
  long long tw_off;
  // Peer destinations (distributed six-step, fused exchange): when npeer > 0 the chunk
  // index (k >> ocl) selects the base pointer peer[k >> ocl] (another rank's receive
  // buffer, mapped over NVLink) instead of out + (k >> ocl) * out_cs.
  int npeer;
  unsigned long long peer[8];
};

}  // namespace fftc
