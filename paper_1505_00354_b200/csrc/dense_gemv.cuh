// The direct DLT / IDLT for few columns: fp64 matrix-vector products over the
// plan's table of P_m(x_k) (dense_gemv.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

struct DenseGemv;

// n even in [256, kDenseMaxN] (8192).
bool dense_gemv_supported(size_t n);
// Builds the table P_m(cos(theta*_kind(k) + delta_k)), k < n/2 (delta: the
// plan's own offsets, device), on `st`.
DenseGemv* dense_gemv_create(size_t n, int kind, const double* delta, cudaStream_t st);
void dense_gemv_destroy(DenseGemv* g);
// out = P in (DLT) / out = (m + 1/2) P^T (w . in) (IDLT); device columns of
// strides ld_in / ld_out; nonfinite (device int, may be null) is set for a
// non-finite input (times w).
void dense_gemv_dlt(const DenseGemv& g, const double* in, size_t ld_in, double* out, size_t ld_out,
                    size_t cols, int* nonfinite, cudaStream_t st);
void dense_gemv_idlt(const DenseGemv& g, const double* in, size_t ld_in, const double* w, double* out,
                     size_t ld_out, size_t cols, int* nonfinite, cudaStream_t st);

}  // namespace flb
