// Generic chirp-z DCT/DST engine and Taylor NDCT (any N, both grid kinds).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

// trig.hpp:55-136 for `batch` device columns (stride ld).
void czt_trig(int op, int kind, size_t n, const double* in, double* out, size_t batch, size_t ld,
              cudaStream_t s);

// ndct.hpp:98-143 literally (kind's own grid and L terms), device pointers.
// in_mult (nullable): per-row factor applied to the input (IDLT weights).
// nonfinite (nullable): device flag set when a term-0 input is not finite.
void czt_ndct(int transpose, int kind, size_t n, int num_terms, const double* delta,
              const double* in, double* out, size_t batch, size_t ld, const double* in_mult,
              int* nonfinite, cudaStream_t s, int l_lo = 0, int l_hi = -1);

}  // namespace flb
