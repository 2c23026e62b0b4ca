// Direct O(N^2) evaluations on the device (the reference's oracle.hpp:19-153
// as GPU kernels). They share no code with the fast
// path (different recurrences, no FFTs), so agreement between the two is an
// independent check at sizes where the CPU oracle is too slow.
#include "common.cuh"
#include "direct.cuh"
#include "launch.cuh"

namespace flb {

namespace {

// oracle.hpp:19-48: sum_n c_n P_n(x_j), three-term recurrence per abscissa
__global__ void eval_legendre_kernel(const double* __restrict__ c, size_t n,
                                     const double* __restrict__ xs, size_t m,
                                     double* __restrict__ out) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const double x = xs[j];
  double p_prev = 1.0;
  double acc = n > 0 ? c[0] : 0.0;
  if (n > 1) {
    double p = x;
    acc += c[1] * p;
    for (size_t q = 1; q + 1 < n; ++q) {
      const double next = ((2.0 * (double)q + 1.0) * x * p - (double)q * p_prev) / ((double)q + 1.0);
      p_prev = p;
      p = next;
      acc += c[q + 1] * p;
    }
  }
  out[j] = acc;
}

// oracle.hpp:52-79: sum_n c_n T_n(x_j)
__global__ void eval_chebyshev_kernel(const double* __restrict__ c, size_t n,
                                      const double* __restrict__ xs, size_t m,
                                      double* __restrict__ out) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const double x = xs[j];
  double t_prev = 1.0;
  double acc = n > 0 ? c[0] : 0.0;
  if (n > 1) {
    double t = x;
    acc += c[1] * t;
    for (size_t q = 1; q + 1 < n; ++q) {
      const double next = 2.0 * x * t - t_prev;
      t_prev = t;
      t = next;
      acc += c[q + 1] * next;
    }
  }
  out[j] = acc;
}

__global__ void domain_kernel(const double* __restrict__ xs, size_t m, int* flag) {
  for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < m;
       j += (size_t)gridDim.x * blockDim.x)
    if (!(fabs(xs[j]) <= 1.0)) atomicOr(flag, 1);
}

// oracle.hpp:84-116: c_m = (m + 1/2) sum_k w_k f_k P_m(x_k). One thread per
// node runs the recurrence over all degrees; each CTA reduces its nodes per
// degree in shared memory and writes one partial row (deterministic order).
constexpr int kIdltNodes = 256;
constexpr int kIdltDeg = 64;  // degrees per shared-memory round

__global__ void __launch_bounds__(kIdltNodes)
    idlt_partial_kernel(const double* __restrict__ f, const double* __restrict__ x,
                        const double* __restrict__ w, size_t n, double* __restrict__ partial) {
  __shared__ double red[kIdltDeg][kIdltNodes / 32];
  const size_t k = blockIdx.x * (size_t)kIdltNodes + threadIdx.x;
  const bool on = k < n;
  const double wf = on ? w[k] * f[k] : 0.0;
  const double xk = on ? x[k] : 0.0;
  double p_prev = 1.0, p = xk;  // P_0, P_1
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (size_t m0 = 0; m0 < n; m0 += kIdltDeg) {
    for (int dm = 0; dm < kIdltDeg; ++dm) {
      const size_t m = m0 + dm;
      double pm;
      if (m == 0) {
        pm = 1.0;
      } else if (m == 1) {
        pm = xk;
      } else {
        // P_m from P_{m-1} = p, P_{m-2} = p_prev (oracle.hpp:103-110 ordering)
        const double a = (2.0 * (double)(m - 1) + 1.0) / ((double)(m - 1) + 1.0);
        const double b = (double)(m - 1) / ((double)(m - 1) + 1.0);
        const double next = a * xk * p - b * p_prev;
        p_prev = p;
        p = next;
        pm = next;
      }
      double v = m < n ? wf * pm : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
      if (lane == 0) red[dm][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < kIdltDeg) {
      const size_t m = m0 + threadIdx.x;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kIdltNodes / 32; ++q) s += red[threadIdx.x][q];
      if (m < n) partial[blockIdx.x * n + m] = s;
    }
    __syncthreads();
  }
}

__global__ void idlt_reduce_kernel(const double* __restrict__ partial, size_t blocks, size_t n,
                                   double* __restrict__ out) {
  const size_t m = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (m >= n) return;
  double s = 0.0;
  for (size_t b = 0; b < blocks; ++b) s += partial[b * n + m];
  out[m] = ((double)m + 0.5) * s;
}

// oracle.hpp:122-153: samples of P_n at m first-kind points, then the
// cosine sums a_k = (2 - delta_k0)/m sum_j s_j cos(k (j+1/2) pi/m).
__global__ void cheb_samples_kernel(size_t n, size_t m, double* __restrict__ samples) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const double x = cos(((double)j + 0.5) * kPi / (double)m);
  if (n == 0) {
    samples[j] = 1.0;
    return;
  }
  double p_prev = 1.0, p = x;
  for (size_t q = 1; q < n; ++q) {
    const double next = ((2.0 * (double)q + 1.0) * x * p - (double)q * p_prev) / ((double)q + 1.0);
    p_prev = p;
    p = next;
  }
  samples[j] = p;
}

__global__ void cheb_coeffs_kernel(size_t n, size_t m, const double* __restrict__ samples,
                                   double* __restrict__ out) {
  const size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (k > n) return;
  double acc = 0.0;
  for (size_t j = 0; j < m; ++j) {
    // cos(k (2j+1) pi / (2m)), phase reduced exactly modulo 4m
    const unsigned long long num = ((unsigned long long)k * (2ull * j + 1ull)) % (4ull * m);
    acc += samples[j] * cospi((double)num / (double)(2 * m));
  }
  out[k] = (k == 0 ? 1.0 : 2.0) / (double)m * acc;
}

unsigned blocks_for(size_t work, int threads) { return (unsigned)((work + threads - 1) / threads); }

}  // namespace

bool direct_domain_ok(const double* xs, size_t m, cudaStream_t s) {
  if (m == 0) return true;
  int* flag = nullptr;
  FLB_CUDA(cudaMallocAsync(&flag, sizeof(int), s));
  FLB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
  domain_kernel<<<sm_count() * 4, 256, 0, s>>>(xs, m, flag);
  note_launch("domain_kernel");
  int h = 0;
  FLB_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  FLB_CUDA(cudaFreeAsync(flag, s));
  FLB_CUDA(cudaStreamSynchronize(s));
  return h == 0;
}

void direct_eval(int chebyshev, const double* c, size_t n, const double* xs, size_t m, double* out,
                 cudaStream_t s) {
  if (m == 0) return;
  if (chebyshev)
    eval_chebyshev_kernel<<<blocks_for(m, 128), 128, 0, s>>>(c, n, xs, m, out);
  else
    eval_legendre_kernel<<<blocks_for(m, 128), 128, 0, s>>>(c, n, xs, m, out);
  note_launch(chebyshev ? "eval_chebyshev_kernel" : "eval_legendre_kernel");
}

void direct_idlt(const double* f, const double* x, const double* w, size_t n, double* out,
                 cudaStream_t s) {
  if (n == 0) return;
  const size_t blocks = (n + kIdltNodes - 1) / kIdltNodes;
  double* partial = nullptr;
  FLB_CUDA(cudaMallocAsync(&partial, blocks * n * sizeof(double), s));
  idlt_partial_kernel<<<(unsigned)blocks, kIdltNodes, 0, s>>>(f, x, w, n, partial);
  note_launch("idlt_partial_kernel");
  idlt_reduce_kernel<<<blocks_for(n, 256), 256, 0, s>>>(partial, blocks, n, out);
  note_launch("idlt_reduce_kernel");
  FLB_CUDA(cudaFreeAsync(partial, s));
}

void direct_cheb_coeffs(size_t n, size_t m, double* out, cudaStream_t s) {
  double* samples = nullptr;
  FLB_CUDA(cudaMallocAsync(&samples, m * sizeof(double), s));
  cheb_samples_kernel<<<blocks_for(m, 128), 128, 0, s>>>(n, m, samples);
  note_launch("cheb_samples_kernel");
  cheb_coeffs_kernel<<<blocks_for(n + 1, 128), 128, 0, s>>>(n, m, samples, out);
  note_launch("cheb_coeffs_kernel");
  FLB_CUDA(cudaFreeAsync(samples, s));
}

}  // namespace flb
