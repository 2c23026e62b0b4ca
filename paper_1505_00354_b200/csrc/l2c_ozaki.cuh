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

// The direct DLT / IDLT as one dense split GEMM per parity (transforms.hpp
// :42-64 evaluated as f = P c and c = D_s P^T D_w f, P_kn = P_n(x_k)): for
// n a multiple of 256 in [512, kDenseMaxN]. The A digits are built from a
// double-double table of P_n(cos theta_k) at the reference's evaluation
// angles theta*_kind(k) + delta_k (delta: the plan's own offsets, device).
constexpr size_t kDenseMaxN = 8192;
bool l2c_dense_supported(size_t n);
L2COzaki* l2c_dense_create(size_t n, int kind, const double* delta, int idlt, cudaStream_t st);
// The table itself: table[m (n/2) + k] = P_m(cos(theta*_kind(k) + delta_k)),
// k < n/2 (double-double, rounded once), n even.
void launch_legendre_table(size_t n, int kind, const double* delta, double* table, cudaStream_t st);
// DLT: out = P in; IDLT: out = (m + 1/2) P^T (w . in) (w: the quadrature
// weights, device). Input / output columns of strides ld_in / ld_out.
// nonfinite (device int, may be null): set when an input column (times w)
// is not finite; that column comes out NaN.
void l2c_dense_apply(const L2COzaki& p, const double* in, size_t ld_in, const double* w,
                     double* out, size_t ld_out, size_t cols, int* nonfinite, cudaStream_t st);

}  // namespace flb
