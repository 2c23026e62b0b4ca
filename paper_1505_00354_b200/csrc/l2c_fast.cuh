// Fast (Toeplitz-Hankel) Legendre <-> Chebyshev conversion for large N.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

struct L2CFast;

// Builds the per-parity low-rank Hankel factors from s = Lambda/Lambda(0)
// (device, n entries). O(n K^2) on the device, K ~ 30-70.
L2CFast* l2c_fast_create(size_t n, const double* s, cudaStream_t st);
void l2c_fast_destroy(L2CFast* f);
int l2c_fast_rank(const L2CFast& f, int parity);

// out = M in (transpose 0) or M^T in (1, optional (m + 1/2) scaling); columns
// of stride ld; in and out must not alias.
// r_lo/r_hi: only the rank terms [r_lo, r_hi) of each parity (a partial
// sum; the rank-parallel multi-GPU DLT splits them over ranks).
void l2c_fast_apply(const L2CFast& f, int transpose, const double* in, double* out, size_t cols,
                    size_t ld, int scale_half, cudaStream_t st, int r_lo = 0, int r_hi = -1);

// Size from which the fast conversion replaces the direct one for few columns.
constexpr size_t kL2CFastMin = size_t(1) << 14;  // 16384: 0.44 ms direct vs TH (C3 sweep)
constexpr size_t kL2CFastMaxCols = 16;

}  // namespace flb
