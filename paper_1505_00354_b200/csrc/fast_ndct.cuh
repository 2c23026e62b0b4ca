// Fused Taylor NDCT on the cheb1 grid for power-of-two N (the hot path).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

struct FastNdct;

// Plan for the nodes `theta` (device, n entries): Taylor expansion about the
// cheb1 angles with min_taylor_terms(cheb1, tol) terms. Returns null when n
// is not a supported power of two.
FastNdct* fast_ndct_create(size_t n, double tol, int kind, const double* theta);
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
