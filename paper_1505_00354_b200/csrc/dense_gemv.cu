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
// m < N, contiguous, 16-byte aligned as N is even): a lane reads the entries
// of two consecutive degrees at once (128-bit loads, 8 entries in flight per
// lane: the 8-byte version reached 2.1 TB/s on the 256 MiB table of N = 8192),
// sums the even degrees (E) and the odd ones (O) separately, and two shuffle
// reductions combine the lanes (fixed order: bit-reproducible). The column
// entries are read by 8-byte loads (any alignment of the caller's pointer).
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
  const double2* row = reinterpret_cast<const double2*>(table_t + k * n);
  const double* cin = in + c0 * ld_in;
  double ev[kCB], od[kCB];
#pragma unroll
  for (int j = 0; j < kCB; ++j) ev[j] = od[j] = 0.0;
  bool bad = false;
  const bool check = k == 0;  // one warp checks every input entry
  constexpr int kU = 4;       // 128-bit table loads in flight per lane
  for (size_t h0 = lane; h0 < r; h0 += 32 * kU) {  // h: degree pair (2h, 2h + 1)
    double2 p[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const size_t h = h0 + 32 * q;
      p[q] = h < r ? __ldg(row + h) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const size_t h = h0 + 32 * q;
      if (h >= r) break;
#pragma unroll
      for (int j = 0; j < kCB; ++j) {
        if (j >= nc) break;
        const double ce = __ldg(cin + j * ld_in + 2 * h), co = __ldg(cin + j * ld_in + 2 * h + 1);
        if (check) bad |= !isfinite(ce) || !isfinite(co);
        ev[j] = __fma_rn(p[q].x, ce, ev[j]);
        od[j] = __fma_rn(p[q].y, co, od[j]);
      }
    }
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
#pragma unroll
  for (int j = 0; j < kCB; ++j) {
    double e = ev[j], o = od[j];
    for (int sh = 16; sh > 0; sh >>= 1) {
      e += __shfl_xor_sync(0xffffffffu, e, sh);
      o += __shfl_xor_sync(0xffffffffu, o, sh);
    }
    if (lane == 0 && j < nc) {
      double* f = out + (c0 + j) * ld_out;
      f[k] = e + o;
      f[n - 1 - k] = e - o;
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

// u_par[k] = w_k f_k +- w_{N-1-k} f_{N-1-k} (k < N/2), per column: [col][2][r]
// (rounded products, then the sum: the reference's (w f)_k +- (w f)_{N-1-k})
__global__ void gemv_idlt_prep_kernel(const double* __restrict__ in, size_t ld_in,
                                      const double* __restrict__ wq, size_t n, size_t cols,
                                      double* __restrict__ u, int* nonfinite) {
  const size_t r = n / 2;
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= r * cols) return;
  const size_t col = i / r, k = i - col * r;
  const double* f = in + col * ld_in;
  const double wa = __dmul_rn(wq[k], f[k]), wbb = __dmul_rn(wq[n - 1 - k], f[n - 1 - k]);
  if (nonfinite && (!isfinite(wa) || !isfinite(wbb))) atomicOr(nonfinite, 1);
  u[(col * 2 + 0) * r + k] = __dadd_rn(wa, wbb);
  u[(col * 2 + 1) * r + k] = __dsub_rn(wa, wbb);
}

// Transposed: one warp per degree m; lanes stride the nodes k (row m of the
// table is contiguous), a shuffle reduction, c_m = (m + 1/2) sum.
// INLINE (short single columns, C1): u is formed from the column as it is
// read, which saves the prep launch and its scratch allocation (N = 1024:
// 31 -> 18 us per call) but repeats the products in every warp (N = 8192:
// 88 -> 120 us, so larger sizes keep the prep pass). The warp of m = 0 then
// checks every input entry.
// VEC: N/2 even, rows 16-byte aligned: 128-bit table loads (two nodes per lane).
template <bool VEC, bool INLINE>
__global__ void __launch_bounds__(32 * kRows) gemv_idlt_kernel(const double* __restrict__ table, size_t n,
                                                               const double* __restrict__ in, size_t ld_in,
                                                               const double* __restrict__ wq,
                                                               const double* __restrict__ uu,
                                                               double* __restrict__ out, size_t ld_out,
                                                               size_t cols, int* nonfinite) {
  const size_t r = n / 2;
  const int lane = threadIdx.x & 31;
  const size_t m = blockIdx.x * (size_t)kRows + (threadIdx.x >> 5);
  if (m >= n) return;
  const size_t c0 = blockIdx.y * (size_t)kCB;
  const int nc = (int)std::min<size_t>(kCB, cols - c0);
  const bool odd = (m & 1) != 0;
  const bool check = INLINE && m == 0;
  bool bad = false;
  const double* row = table + m * r;
  const double* fin = INLINE ? in + c0 * ld_in : nullptr;
  const double* up = INLINE ? nullptr : uu + (c0 * 2 + (odd ? 1 : 0)) * r;  // column j: + 2 j r
  double acc[kCB];
#pragma unroll
  for (int j = 0; j < kCB; ++j) acc[j] = 0.0;
  // u_k of column j: rounded products, then the sum (as the reference forms (w f)_k first)
  auto u_of = [&](int j, size_t k, double wk, double wb) {
    if constexpr (!INLINE) return __ldg(up + 2 * (size_t)j * r + k);
    const double a = __ldg(fin + j * ld_in + k), b = __ldg(fin + j * ld_in + (n - 1 - k));
    const double wa = __dmul_rn(wk, a), wbb = __dmul_rn(wb, b);
    if (check) bad |= !isfinite(wa) || !isfinite(wbb);
    return odd ? __dsub_rn(wa, wbb) : __dadd_rn(wa, wbb);
  };
  if constexpr (VEC) {
    constexpr int kU = 4;
    const double2* row2 = reinterpret_cast<const double2*>(row);
    double acc2[kCB];
#pragma unroll
    for (int j = 0; j < kCB; ++j) acc2[j] = 0.0;
    for (size_t h0 = lane; h0 < r / 2; h0 += 32 * kU) {  // h: node pair (2h, 2h + 1)
      double2 p[kU];
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const size_t h = h0 + 32 * q;
        p[q] = h < r / 2 ? __ldg(row2 + h) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < kU; ++q) {
        const size_t h = h0 + 32 * q;
        if (h >= r / 2) break;
        const size_t k = 2 * h;
        const double wk0 = INLINE ? __ldg(wq + k) : 0.0, wb0 = INLINE ? __ldg(wq + (n - 1 - k)) : 0.0;
        const double wk1 = INLINE ? __ldg(wq + k + 1) : 0.0, wb1 = INLINE ? __ldg(wq + (n - 2 - k)) : 0.0;
#pragma unroll
        for (int j = 0; j < kCB; ++j) {
          if (j >= nc) break;
          acc[j] = __fma_rn(p[q].x, u_of(j, k, wk0, wb0), acc[j]);
          acc2[j] = __fma_rn(p[q].y, u_of(j, k + 1, wk1, wb1), acc2[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kCB; ++j) acc[j] += acc2[j];
  } else {
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
        const double wk = INLINE ? __ldg(wq + k) : 0.0, wb = INLINE ? __ldg(wq + (n - 1 - k)) : 0.0;
#pragma unroll
        for (int j = 0; j < kCB; ++j) {
          if (j >= nc) break;
          acc[j] = __fma_rn(p[q], u_of(j, k, wk, wb), acc[j]);
        }
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
  const size_t n = g.n, r = n / 2;
  const dim3 grid((unsigned)((n + kRows - 1) / kRows), (unsigned)((cols + kCB - 1) / kCB));
  const bool vec = r % 2 == 0;
  if (n <= 2048 && cols <= (size_t)kCB) {  // short single columns: no prep pass
    auto kern = vec ? gemv_idlt_kernel<true, true> : gemv_idlt_kernel<false, true>;
    kern<<<grid, 32 * kRows, 0, st>>>(g.table, n, in, ld_in, w, nullptr, out, ld_out, cols, nonfinite);
    note_launch("gemv_idlt_kernel");
    return;
  }
  double* u = nullptr;
  FLB_CUDA(cudaMallocAsync(&u, 2 * r * cols * sizeof(double), st));
  gemv_idlt_prep_kernel<<<(unsigned)((r * cols + 255) / 256), 256, 0, st>>>(in, ld_in, w, n, cols, u,
                                                                             nonfinite);
  note_launch("gemv_idlt_prep_kernel");
  auto kern = vec ? gemv_idlt_kernel<true, false> : gemv_idlt_kernel<false, false>;
  kern<<<grid, 32 * kRows, 0, st>>>(g.table, n, nullptr, 0, nullptr, u, out, ld_out, cols, nonfinite);
  note_launch("gemv_idlt_kernel");
  cudaFreeAsync(u, st);
}

}  // namespace flb
