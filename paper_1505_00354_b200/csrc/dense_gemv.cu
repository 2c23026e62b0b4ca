// The direct DLT / IDLT for few columns (<= 16) at N <= 8192: f = P c and
// c = (m + 1/2) P^T (w . f) as fp64 matrix-vector products over the plan's
// table P_m(x_k) (double-double at the reference's evaluation angles
// theta*_kind(k) + delta_k, rounded once: the table the batched direct method
// splits into int8 digits, l2c_ozaki.cu), kept in both layouts so that every
// dot product streams a contiguous row. transforms.hpp:42-64 evaluates the
// same maps as conversion + NDCT (two latency-bound kernels for one column: a
// single CTA runs all NDCT terms); here one pass over the table (N^2/2
// doubles: 4 MiB at 1024, L2-resident; 256 MiB at 8192).
//
//   E_k = sum_{m even} P_m(x_k) c_m,  O_k = sum_{m odd} P_m(x_k) c_m   (k < N/2)
//   f_k = E_k + O_k,  f_{N-1-k} = E_k - O_k        (P_m(-x) = (-1)^m P_m(x))
//   c_m = (m + 1/2) sum_{k < N/2} P_m(x_k) w_k (f_k + (-1)^m f_{N-1-k})
#include "dense_gemv.cuh"

#include <algorithm>

#include "common.cuh"
#include "launch.cuh"
#include "l2c_ozaki.cuh"

namespace flb {
namespace {

constexpr int kCB = 4;      // columns per pass (each table entry read once per pass)
constexpr int kRows = 8;    // table rows (one per warp) per CTA

// Forward: one warp per node k over the transposed table (row k = P_m(x_k),
// m < N, contiguous): lanes stride the degrees, so even lanes sum the even
// degrees (E) and odd lanes the odd ones (O); parity-preserving shuffles
// combine them (fixed order: bit-reproducible).
__global__ void __launch_bounds__(32 * kRows) gemv_dlt_kernel(const double* __restrict__ table_t, size_t n,
                                                              const double* __restrict__ in, size_t ld_in,
                                                              double* __restrict__ out, size_t ld_out,
                                                              size_t cols, int* nonfinite) {
  const size_t r = n / 2;
  const int lane = threadIdx.x & 31;
  const size_t k = blockIdx.x * (size_t)kRows + (threadIdx.x >> 5);
  if (k >= r) return;
  const size_t c0 = blockIdx.y * (size_t)kCB;
  const int nc = (int)std::min<size_t>(kCB, cols - c0);
  const double* row = table_t + k * n;
  const double* cin = in + c0 * ld_in;
  double acc[kCB];
#pragma unroll
  for (int j = 0; j < kCB; ++j) acc[j] = 0.0;
  bool bad = false;
  const bool check = k == 0;  // one warp checks every input entry
  constexpr int kU = 8;       // table entries in flight per lane
  for (size_t m0 = lane; m0 < n; m0 += 32 * kU) {
    double p[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const size_t m = m0 + 32 * q;
      p[q] = m < n ? __ldg(row + m) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const size_t m = m0 + 32 * q;
      if (m >= n) break;
#pragma unroll
      for (int j = 0; j < kCB; ++j) {
        if (j >= nc) break;
        const double cm = __ldg(cin + j * ld_in + m);
        if (check) bad |= !isfinite(cm);
        acc[j] = __fma_rn(p[q], cm, acc[j]);
      }
    }
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
#pragma unroll
  for (int j = 0; j < kCB; ++j) {
    double v = acc[j];
    for (int o = 16; o >= 2; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);  // lane parity kept
    const double odd = __shfl_sync(0xffffffffu, v, 1);
    if (lane == 0 && j < nc) {
      double* f = out + (c0 + j) * ld_out;
      f[k] = v + odd;
      f[n - 1 - k] = v - odd;
    }
  }
}

// table_t[k][m] = table[m][k] (32 x 32 tiles through shared memory)
__global__ void gemv_transpose_kernel(const double* __restrict__ table, size_t n, double* __restrict__ table_t) {
  __shared__ double tile[32][33];
  const size_t r = n / 2;
  const size_t m0 = blockIdx.y * (size_t)32, k0 = blockIdx.x * (size_t)32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const size_t m = m0 + i, k = k0 + threadIdx.x;
    if (m < n && k < r) tile[i][threadIdx.x] = table[m * r + k];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const size_t k = k0 + i, m = m0 + threadIdx.x;
    if (m < n && k < r) table_t[k * n + m] = tile[threadIdx.x][i];
  }
}

// Transposed: one warp per degree m; lanes stride the nodes k (row m of the
// table is contiguous), a shuffle reduction, c_m = (m + 1/2) sum. The input
// u_par[k] = w_k f_k +- w_{N-1-k} f_{N-1-k} (the reference's (w f)_k +-
// (w f)_{N-1-k}) is formed from the column as it is read (the values are
// L1 / L2 hits beside the table stream; a separate pass cost an allocation
// and a launch per call). The warp of m = 0 checks every input entry.
__global__ void __launch_bounds__(32 * kRows) gemv_idlt_kernel(const double* __restrict__ table, size_t n,
                                                               const double* __restrict__ in, size_t ld_in,
                                                               const double* __restrict__ wq,
                                                               double* __restrict__ out, size_t ld_out,
                                                               size_t cols, int* nonfinite) {
  const size_t r = n / 2;
  const int lane = threadIdx.x & 31;
  const size_t m = blockIdx.x * (size_t)kRows + (threadIdx.x >> 5);
  if (m >= n) return;
  const size_t c0 = blockIdx.y * (size_t)kCB;
  const int nc = (int)std::min<size_t>(kCB, cols - c0);
  const bool odd = (m & 1) != 0;
  const bool check = m == 0;
  bool bad = false;
  const double* row = table + m * r;
  const double* fin = in + c0 * ld_in;
  double acc[kCB];
#pragma unroll
  for (int j = 0; j < kCB; ++j) acc[j] = 0.0;
  constexpr int kU = 8;
  for (size_t k0 = lane; k0 < r; k0 += 32 * kU) {
    double p[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const size_t k = k0 + 32 * q;
      p[q] = k < r ? __ldg(row + k) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const size_t k = k0 + 32 * q;
      if (k >= r) break;
      const double wk = __ldg(wq + k), wb = __ldg(wq + (n - 1 - k));
#pragma unroll
      for (int j = 0; j < kCB; ++j) {
        if (j >= nc) break;
        const double a = __ldg(fin + j * ld_in + k), b = __ldg(fin + j * ld_in + (n - 1 - k));
        // rounded products, then the sum (as the reference forms (w f)_k first)
        const double wa = __dmul_rn(wk, a), wbb = __dmul_rn(wb, b);
        if (check) bad |= !isfinite(wa) || !isfinite(wbb);
        const double u = odd ? __dsub_rn(wa, wbb) : __dadd_rn(wa, wbb);
        acc[j] = __fma_rn(p[q], u, acc[j]);
      }
    }
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
#pragma unroll
  for (int j = 0; j < kCB; ++j) {
    double v = acc[j];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && j < nc) out[(c0 + j) * ld_out + m] = ((double)m + 0.5) * v;
  }
}

}  // namespace

struct DenseGemv {
  size_t n = 0;
  double* table = nullptr;    // [m][k]: P_m(x_k), k < n/2 (rows: the IDLT's dot products)
  double* table_t = nullptr;  // [k][m] (rows: the DLT's)
};

bool dense_gemv_supported(size_t n) { return n % 2 == 0 && n >= 256 && n <= kDenseMaxN; }

DenseGemv* dense_gemv_create(size_t n, int kind, const double* delta, cudaStream_t st) {
  if (!dense_gemv_supported(n)) fail(FL_INVALID_ARGUMENT, "dense_gemv: unsupported size");
  auto* g = new DenseGemv;
  g->n = n;
  FLB_CUDA(cudaMalloc(&g->table, n * (n / 2) * sizeof(double)));
  FLB_CUDA(cudaMalloc(&g->table_t, n * (n / 2) * sizeof(double)));
  launch_legendre_table(n, kind, delta, g->table, st);
  gemv_transpose_kernel<<<dim3((unsigned)((n / 2 + 31) / 32), (unsigned)((n + 31) / 32)), dim3(32, 8), 0, st>>>(
      g->table, n, g->table_t);
  note_launch("gemv_transpose_kernel");
  return g;
}

void dense_gemv_destroy(DenseGemv* g) {
  if (!g) return;
  if (g->table) cudaFree(g->table);
  if (g->table_t) cudaFree(g->table_t);
  delete g;
}

void dense_gemv_dlt(const DenseGemv& g, const double* in, size_t ld_in, double* out, size_t ld_out,
                    size_t cols, int* nonfinite, cudaStream_t st) {
  if (cols == 0) return;
  const size_t r = g.n / 2;
  const dim3 grid((unsigned)((r + kRows - 1) / kRows), (unsigned)((cols + kCB - 1) / kCB));
  gemv_dlt_kernel<<<grid, 32 * kRows, 0, st>>>(g.table_t, g.n, in, ld_in, out, ld_out, cols, nonfinite);
  note_launch("gemv_dlt_kernel");
}

void dense_gemv_idlt(const DenseGemv& g, const double* in, size_t ld_in, const double* w, double* out,
                     size_t ld_out, size_t cols, int* nonfinite, cudaStream_t st) {
  if (cols == 0) return;
  const size_t n = g.n;
  const dim3 grid((unsigned)((n + kRows - 1) / kRows), (unsigned)((cols + kCB - 1) / kCB));
  gemv_idlt_kernel<<<grid, 32 * kRows, 0, st>>>(g.table, n, in, ld_in, w, out, ld_out, cols, nonfinite);
  note_launch("gemv_idlt_kernel");
}

}  // namespace flb
