// Fused Taylor NDCT on the cheb1 grid for power-of-two N (the hot path).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

struct FastNdct;

// Plan for the node offsets `delta` (device, n entries: delta_theta of grid
// `kind`, quadrature.hpp:147-158): the nodes evaluated about the cheb1
// angles (delta' = delta + the exact grid offset) by the Chebyshev
// (Jacobi-Anger) expansion to `tol`. Returns null when n is not a supported
// power of two.
FastNdct* fast_ndct_create(size_t n, double tol, int kind, const double* delta);
// The same evaluation for a caller's offsets (the free-function NDCT, and
// with delta = null the chebstar DCT/DST): returns null unless the literal
// L-term evaluation (ndct.hpp:98-143) is exact to fp64 rounding (so both agree
// to rounding) and the expansion converges (M <= 30 terms to 2^-52 at the
// measured max |N delta'|). swap: the sine flavour. Buffers are stream-ordered
// on s; the call synchronises s once (the max |delta| reduction).
FastNdct* fast_ndct_create_bessel(size_t n, int kind, const double* delta, int num_terms,
                                  int swap, cudaStream_t s);
// A literal cheb1 plan with caller-owned device delta_theta (fl_ndct).
bool fast_ndct_literal_ok(size_t n, int kind);
FastNdct* fast_ndct_create_literal(size_t n, int kind, int num_terms, const double* delta,
                                   cudaStream_t s);
void fast_ndct_destroy(FastNdct* p);

// Power-of-two cheb1 dct_iii / dst_iii / *_transpose (trig.hpp) through the
// same fused kernels with one unscaled term.
bool fast_trig_ok(size_t n, int kind);
void fast_trig(int op, size_t n, const double* in, double* out, size_t batch, size_t ld,
               cudaStream_t s);
// The chebstar ones at power-of-two N through the Chebyshev expansion.
bool fast_trig_bessel_ok(size_t n, int kind);
void fast_trig_bessel(int op, size_t n, const double* in, double* out, size_t batch, size_t ld,
                      cudaStream_t s);

struct FastNdctHolder {
  FastNdct* p = nullptr;
  ~FastNdctHolder() {
    if (p) fast_ndct_destroy(p);
  }
};

// forward: out = NDCT(in); transpose: out = NDCT^T(in_mult . in).
// nonfinite: device flag, set when a (weighted) input is not finite.
// Terms [l_lo, l_hi) only (l_hi < 0: all): a partial Taylor sum, used by the
// term-parallel multi-GPU DLT (only for N > 8192, the multi-pass path).
void fast_ndct_run(const FastNdct& p, int transpose, const double* in, size_t ld_in, double* out,
                   size_t ld_out, size_t batch, const double* in_mult, int* nonfinite,
                   cudaStream_t s, int l_lo = 0, int l_hi = -1);
int fast_ndct_terms(const FastNdct& p);
// Transforms per column of fast_ndct_run for N <= 8192 (the Chebyshev
// expansion's term count when it is in use, else the Taylor count).
int fast_ndct_dlt_terms(const FastNdct& p);

}  // namespace flb
