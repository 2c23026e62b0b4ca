// Kernel-launch bookkeeping and the internal launcher declarations shared by
// the translation units of libfastleg_b200.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

// Counts every kernel this library launches (fl_kernel_launch_count) and
// turns a launch failure into an Error.
void note_launch(const char* name);

// nodes.cu
double lambda_value_host(unsigned long long z);
void launch_nodes(size_t n, double* theta, double* x, double* w, cudaStream_t s);
void launch_reference_grid(size_t n, int kind, const double* theta, double* theta_star,
                           double* delta, cudaStream_t s);
void launch_lambda(size_t max_index, double* table, cudaStream_t s);

}  // namespace flb
