// Legendre <-> Chebyshev conversion as an exact-integer split GEMM on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

struct L2COzaki;

// Shapes the split GEMM handles: n a multiple of 256 in [512, 2^16].
bool l2c_ozaki_supported(size_t n);

// Slices of the parity blocks of M (transpose = 0) or M^T (1, rows times
// (m + 1/2) when scale_half) built from the scaled Lambda table s (device).
L2COzaki* l2c_ozaki_create(size_t n, const double* s, int transpose, int scale_half,
                           cudaStream_t st);
void l2c_ozaki_destroy(L2COzaki* p);

// out = M in (or (m + 1/2) M^T in), `cols` device columns of stride ld.
void l2c_ozaki_apply(const L2COzaki& p, const double* in, double* out, size_t cols, size_t ld,
                     cudaStream_t st);

}  // namespace flb
