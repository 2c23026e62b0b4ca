// Direct O(N^2) evaluations on the device (oracle.hpp:19-153).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

bool direct_domain_ok(const double* xs, size_t m, cudaStream_t s);  // all |x| <= 1
void direct_eval(int chebyshev, const double* c, size_t n, const double* xs, size_t m, double* out,
                 cudaStream_t s);
void direct_idlt(const double* f, const double* x, const double* w, size_t n, double* out,
                 cudaStream_t s);
void direct_cheb_coeffs(size_t n, size_t m, double* out, cudaStream_t s);

}  // namespace flb
