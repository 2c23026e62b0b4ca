// Legendre -> Chebyshev conversion M c and its transpose M^T v, direct.
//
// Replaces conversion.hpp:100-140. With s_j = Lambda(j)/Lambda(0)
// (conversion.hpp:88-94) the upper-triangular, parity-split matrix is
//   M_{k, k+2j} = (2 - delta_{k0}) s_j s_{k+j}
// so
//   forward   (conversion.hpp:106-111): chat_k = (2 - delta_k0) sum_{k+2j<N} s_j s_{k+j} c_{k+2j}
//   transpose (conversion.hpp:126-133): out_m = 2 sum_{2j<m} s_j s_{m-j} v_{m-2j}
//                                              + [m even] s_{m/2} s_{m-m/2} v_0
// Batched over columns. The triangle of each parity class is tiled: a CTA
// owns TK output rows x TC columns; the s-table and input tiles stream
// through shared memory and each thread accumulates a 4 x 4 register block
// (a triangular fp64 GEMM, FMA-pipe bound; SURVEY.md 8d gives N/2 flop/coef).
#include "common.cuh"
#include "launch.cuh"
#include "leg2cheb.cuh"

namespace flb {

namespace {

__global__ void scaled_lambda_kernel(const double* __restrict__ table, double* __restrict__ s,
                                     size_t count) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j < count) s[j] = table[j] / table[0];  // conversion.hpp:93
}

// ---------------------------------------------------------------------------
// Tiled kernel. Parity class p in {0,1}: rows k = 2a + p, inputs n = 2b + p,
// b >= a, entry s_{b-a} s_{a+b+p}. Row tile [a0, a0+TA), column tile
// [c0, c0+TC). Inner dimension b runs from a0 to the end in chunks of TB.
// ---------------------------------------------------------------------------
constexpr int TA = 64;   // rows (per parity) per CTA
constexpr int TC = 64;   // columns per CTA
constexpr int TB = 16;   // inner chunk
constexpr int RA = 4;    // rows per thread
constexpr int RC = 4;    // columns per thread
constexpr int THREADS = (TA / RA) * (TC / RC);  // 256

__global__ void __launch_bounds__(THREADS)
    leg2cheb_fwd_tiled(const double* __restrict__ s, const double* __restrict__ in,
                       double* __restrict__ out, size_t n, size_t cols, size_t ld) {
  const int p = blockIdx.z;
  const size_t nrows = (n + 1 - p) / 2;   // rows of this parity
  const size_t a0 = (size_t)blockIdx.x * TA;
  const size_t c0 = (size_t)blockIdx.y * TC;
  if (a0 >= nrows) return;
  __shared__ double Ms[TB][TA + 1];  // M[a][b] for the chunk, transposed
  __shared__ double Cs[TB][TC + 1];  // inputs c[2b+p] for the chunk
  const int tx = threadIdx.x % (TC / RC), ty = threadIdx.x / (TC / RC);
  double acc[RA][RC];
#pragma unroll
  for (int i = 0; i < RA; ++i)
#pragma unroll
    for (int j = 0; j < RC; ++j) acc[i][j] = 0.0;
  for (size_t b0 = a0; b0 < nrows; b0 += TB) {
    // M tile: a in [a0, a0+TA), b in [b0, b0+TB)
    for (int i = threadIdx.x; i < TA * TB; i += THREADS) {
      const int aa = i / TB, bb = i % TB;
      const size_t a = a0 + aa, b = b0 + bb;
      double m = 0.0;
      if (b >= a && b < nrows && a < nrows) m = s[b - a] * s[a + b + p];
      Ms[bb][aa] = m;
    }
    // C tile: rows n = 2b+p, columns c0..c0+TC
    for (int i = threadIdx.x; i < TB * TC; i += THREADS) {
      const int bb = i % TB, cc = i / TB;
      const size_t b = b0 + bb, col = c0 + cc;
      Cs[bb][cc] = (b < nrows && col < cols) ? in[col * ld + 2 * b + p] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int bb = 0; bb < TB; ++bb) {
      double mv[RA], cv[RC];
#pragma unroll
      for (int i = 0; i < RA; ++i) mv[i] = Ms[bb][ty + i * (TA / RA)];
#pragma unroll
      for (int j = 0; j < RC; ++j) cv[j] = Cs[bb][tx + j * (TC / RC)];
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int j = 0; j < RC; ++j) acc[i][j] = fma(mv[i], cv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RA; ++i) {
    const size_t a = a0 + ty + i * (TA / RA);
    if (a >= nrows) continue;
    const size_t k = 2 * a + p;
    const double pref = k == 0 ? 1.0 : 2.0;
#pragma unroll
    for (int j = 0; j < RC; ++j) {
      const size_t col = c0 + tx + j * (TC / RC);
      if (col < cols) out[col * ld + k] = pref * acc[i][j];
    }
  }
}

// M^T: out_m (m = 2b + p) = sum_{a <= b} pref_{2a+p} s_{b-a} s_{a+b+p} v_{2a+p}
// (pref = 1 for row k = 0, else 2), optionally times (m + 1/2) (the IDLT's
// D_s, transforms.hpp:62).
__global__ void __launch_bounds__(THREADS)
    leg2cheb_tr_tiled(const double* __restrict__ s, const double* __restrict__ in,
                      double* __restrict__ out, size_t n, size_t cols, size_t ld, int scale_half) {
  const int p = blockIdx.z;
  const size_t nrows = (n + 1 - p) / 2;
  const size_t b0t = (size_t)blockIdx.x * TA;  // output tile (indexed by b)
  const size_t c0 = (size_t)blockIdx.y * TC;
  if (b0t >= nrows) return;
  __shared__ double Ms[TB][TA + 1];  // M[a][b] chunk over a
  __shared__ double Vs[TB][TC + 1];
  const int tx = threadIdx.x % (TC / RC), ty = threadIdx.x / (TC / RC);
  double acc[RA][RC];
#pragma unroll
  for (int i = 0; i < RA; ++i)
#pragma unroll
    for (int j = 0; j < RC; ++j) acc[i][j] = 0.0;
  const size_t a_end = b0t + TA < nrows ? b0t + TA : nrows;  // a <= b < b0t + TA
  for (size_t a0 = 0; a0 < a_end; a0 += TB) {
    for (int i = threadIdx.x; i < TA * TB; i += THREADS) {
      const int bb = i / TB, aa = i % TB;
      const size_t b = b0t + bb, a = a0 + aa;
      double m = 0.0;
      if (a <= b && b < nrows) {
        const double pref = (2 * a + p) == 0 ? 1.0 : 2.0;
        m = pref * (s[b - a] * s[a + b + p]);
      }
      Ms[aa][bb] = m;
    }
    for (int i = threadIdx.x; i < TB * TC; i += THREADS) {
      const int aa = i % TB, cc = i / TB;
      const size_t a = a0 + aa, col = c0 + cc;
      Vs[aa][cc] = (a < nrows && col < cols) ? in[col * ld + 2 * a + p] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int aa = 0; aa < TB; ++aa) {
      double mv[RA], vv[RC];
#pragma unroll
      for (int i = 0; i < RA; ++i) mv[i] = Ms[aa][ty + i * (TA / RA)];
#pragma unroll
      for (int j = 0; j < RC; ++j) vv[j] = Vs[aa][tx + j * (TC / RC)];
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int j = 0; j < RC; ++j) acc[i][j] = fma(mv[i], vv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RA; ++i) {
    const size_t b = b0t + ty + i * (TA / RA);
    if (b >= nrows) continue;
    const size_t m = 2 * b + p;
    const double sc = scale_half ? (double)m + 0.5 : 1.0;
#pragma unroll
    for (int j = 0; j < RC; ++j) {
      const size_t col = c0 + tx + j * (TC / RC);
      if (col < cols) out[col * ld + m] = sc * acc[i][j];
    }
  }
}

}  // namespace

void scaled_lambda(const double* table, double* s, size_t count, cudaStream_t st) {
  if (count == 0) return;
  scaled_lambda_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(table, s, count);
  note_launch("scaled_lambda_kernel");
}

void leg2cheb_direct(int transpose, size_t n, const double* s, const double* in, double* out,
                     size_t cols, size_t ld, int scale_half, cudaStream_t st) {
  if (n == 0 || cols == 0) return;
  const size_t rows = (n + 1) / 2;
  for (size_t c0 = 0; c0 < cols; c0 += (size_t)65535 * TC) {
    const size_t nc = cols - c0 < (size_t)65535 * TC ? cols - c0 : (size_t)65535 * TC;
    dim3 grid((unsigned)((rows + TA - 1) / TA), (unsigned)((nc + TC - 1) / TC), n > 1 ? 2 : 1);
    if (transpose)
      leg2cheb_tr_tiled<<<grid, THREADS, 0, st>>>(s, in + c0 * ld, out + c0 * ld, n, nc, ld,
                                                  scale_half);
    else
      leg2cheb_fwd_tiled<<<grid, THREADS, 0, st>>>(s, in + c0 * ld, out + c0 * ld, n, nc, ld);
    note_launch(transpose ? "leg2cheb_tr_tiled" : "leg2cheb_fwd_tiled");
  }
}

}  // namespace flb
