// Direct Legendre <-> Chebyshev conversion kernels (conversion.hpp:100-140).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

// s_j = table[j] / table[0] for j < count (conversion.hpp:88-94)
void scaled_lambda(const double* table, double* s, size_t count, cudaStream_t st);

// out = M in (transpose = 0) or M^T in (1, optionally times (m + 1/2)),
// `cols` device columns of stride ld. in and out must not alias.
void leg2cheb_direct(int transpose, size_t n, const double* s, const double* in, double* out,
                     size_t cols, size_t ld, int scale_half, cudaStream_t st);

}  // namespace flb
