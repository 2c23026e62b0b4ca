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

// ---------------------------------------------------------------------------
// fp64 tensor-core version (mma.sync.m8n8k4.f64, DMMA). One CTA owns 32 rows
// of BOTH parity classes (output rows [2 a0, 2 a0 + 64), contiguous) x 128
// columns; 8 warps, warp w computes parity w & 1, columns (w >> 1) * 32 + [0, 32)
// as a 4 x 4 grid of 8 x 8 accumulator tiles. The inner dimension streams in
// chunks of 16 per parity: the M chunk is generated from the s table into
// shared memory, the input chunk (rows [2 b0, 2 b0 + 32) of 128 columns, both
// parities) is prefetched into registers one chunk ahead and split by parity
// on the way into shared memory. The epilogue stages the 64 x 128 output
// tile in shared memory and writes whole column segments (coalesced).
//   forward  : A[a][b] = s_{b-a} s_{a+b+p}           (b >= a),  row scale 1 | 2
//   transpose: A[b][a] = pref_{2a+p} s_{b-a} s_{a+b+p} (a <= b), row scale (m + 1/2) opt.
// ---------------------------------------------------------------------------
namespace mma {
constexpr int RA = 32;        // rows per parity per CTA
constexpr int CT = 128;       // columns per CTA
constexpr int KB = 16;        // inner chunk per parity
constexpr int LDA = KB + 4;   // 160 B rows: 8 rows x 32 B hit distinct bank groups per phase
constexpr int LDB = KB + 4;   // input chunk stored column-major [col][k], same 160 B rows
constexpr int THREADS = 256;
constexpr int SM_A = 2 * RA * LDA;   // doubles
constexpr int SM_B = 2 * CT * LDB;   // doubles
constexpr int LDO = 2 * RA + 2;      // epilogue tile: [CT][2 RA] (+2 pad)
constexpr int SM_O = CT * LDO;
constexpr int SMEM_DOUBLES = 2 * (SM_A + SM_B) > SM_O ? 2 * (SM_A + SM_B) : SM_O;
}  // namespace mma

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <bool TR>
__global__ void __launch_bounds__(mma::THREADS, 2)
    leg2cheb_mma_kernel(const double* __restrict__ s, const double* __restrict__ in,
                        double* __restrict__ out, size_t n, size_t cols, size_t ld,
                        int scale_half) {
  constexpr int RA = mma::RA, CT = mma::CT, KB = mma::KB, LDA = mma::LDA, LDB = mma::LDB;
  constexpr int THREADS = mma::THREADS, SM_A = mma::SM_A, SM_B = mma::SM_B, LDO = mma::LDO;
  extern __shared__ double sm[];
  double* As = sm;               // [stage][parity][RA][LDA]
  double* Bs = sm + 2 * SM_A;    // [stage][parity][CT][LDB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wp = warp & 1, wc = (warp >> 1) * 32;
  const size_t a0 = (size_t)blockIdx.x * RA;
  const size_t c0 = (size_t)blockIdx.y * CT;
  const size_t nr[2] = {(n + 1) / 2, n / 2};  // rows per parity
  if (a0 >= nr[0]) return;
  // inner range (union over both parities), chunk aligned
  size_t k_begin, k_end;
  if (!TR) {
    k_begin = a0 - (a0 % KB);
    k_end = nr[0];
  } else {
    k_begin = 0;
    k_end = a0 + RA < nr[0] ? a0 + RA : nr[0];
  }
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // register prefetch of one input chunk: 8 x double2 (rows 2b0..2b0+31, 128 cols)
  double2 pre[8];
  auto load_b = [&](size_t b0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = tid + THREADS * i;
      const int col = idx >> 4, pr = idx & 15;
      const size_t b = b0 + pr, gc = c0 + col;
      double2 v = make_double2(0.0, 0.0);
      if (gc < cols) {
        const double* src = in + gc * ld + 2 * b;
        if (2 * b + 1 < n)
          v = __ldg(reinterpret_cast<const double2*>(src));
        else if (2 * b < n)
          v.x = __ldg(src);
      }
      pre[i] = v;
    }
  };
  auto store_b = [&](int stg) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = tid + THREADS * i;
      const int col = idx >> 4, pr = idx & 15;
      Bs[stg * SM_B + (0 * CT + col) * LDB + pr] = pre[i].x;
      Bs[stg * SM_B + (1 * CT + col) * LDB + pr] = pre[i].y;
    }
  };
  double preA[4];
  auto calc_a = [&](size_t b0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + THREADS * i;
      const int p = idx >> 9, r = (idx >> 4) & 31, kk = idx & 15;
      const size_t row = a0 + r, inner = b0 + kk;
      double v = 0.0;
      if (!TR) {
        if (inner >= row && inner < nr[p]) v = s[inner - row] * s[row + inner + p];
      } else {
        if (inner <= row && row < nr[p]) {
          const double pref = (2 * inner + p) == 0 ? 1.0 : 2.0;
          v = pref * (s[row - inner] * s[row + inner + p]);
        }
      }
      preA[i] = v;
    }
  };
  auto store_a = [&](int stg) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + THREADS * i;
      const int p = idx >> 9, r = (idx >> 4) & 31, kk = idx & 15;
      As[stg * SM_A + (p * RA + r) * LDA + kk] = preA[i];
    }
  };

  // two shared-memory stages: chunk c is multiplied from stage c & 1 while
  // chunk c+1 (prefetched into registers during the MMAs) fills the other one,
  // so one barrier per chunk separates them
  load_b(k_begin);
  calc_a(k_begin);
  store_b(0);
  store_a(0);
  __syncthreads();
  int stg = 0;
  for (size_t b0 = k_begin; b0 < k_end; b0 += KB) {
    const bool more = b0 + KB < k_end;
    if (more) {
      load_b(b0 + KB);
      calc_a(b0 + KB);
    }
    const double* Ap = As + stg * SM_A + wp * RA * LDA;
    const double* Bp = Bs + stg * SM_B + wp * CT * LDB;
#pragma unroll
    for (int ks = 0; ks < KB; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Ap[(8 * i + (lane >> 2)) * LDA + ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bp[(wc + 8 * j + (lane >> 2)) * LDB + ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j], af[i], bf[j]);
    }
    if (more) {
      store_b(stg ^ 1);
      store_a(stg ^ 1);
    }
    __syncthreads();
    stg ^= 1;
  }
  __syncthreads();
  // epilogue: O[col][k_local], k_local = 2 a + p in [0, 64)
  double* O = sm;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = 8 * i + (lane >> 2);
      const int cl = wc + 8 * j + 2 * (lane & 3);
      const int kl = 2 * r + wp;
      O[cl * LDO + kl] = acc[i][j][0];
      O[(cl + 1) * LDO + kl] = acc[i][j][1];
    }
  __syncthreads();
  const size_t k0 = 2 * a0;
  for (int idx = tid; idx < CT * 2 * RA; idx += THREADS) {
    const int cl = idx >> 6, kl = idx & 63;
    const size_t gc = c0 + cl, k = k0 + kl;
    if (gc >= cols || k >= n) continue;
    double v = O[cl * LDO + kl];
    if (!TR)
      v = (k == 0 ? 1.0 : 2.0) * v;
    else if (scale_half)
      v = ((double)k + 0.5) * v;
    out[gc * ld + k] = v;
  }
}

// ---------------------------------------------------------------------------
// Few columns (single vectors up to large N): a tiled matrix-vector product.
// A CTA owns TK consecutive rows of one parity and one column and streams the
// inner index in chunks of KC through shared memory: the Toeplitz factor
// s_{|row - inner|} and the Hankel factor s_{row + inner + p} are staged as
// two zero-padded windows, the input chunk (pref folded in for M^T) as a
// third. Each thread owns RB consecutive rows and slides two RB-register
// windows along the inner index: per inner step 2 new s values + 1 input
// (3 shared loads, 2 broadcast-free) feed RB multiply-adds.
// ---------------------------------------------------------------------------
namespace mv {
constexpr int RB = 8;                 // rows per thread
constexpr int THREADS = 128;
constexpr int TK = RB * THREADS;      // rows per CTA (1024)
constexpr int KC = 256;               // inner chunk
}  // namespace mv

// RB rows per thread x NT threads per CTA (TK = RB NT rows per CTA): the
// default 8 x 128, and 2 x 32 for short vectors (N <= 8192), where the
// default gives one CTA per parity and a 27 us latency at N = 1024.
template <bool TR, int RB = mv::RB, int NT = mv::THREADS>
__global__ void __launch_bounds__(NT)
    leg2cheb_mv_kernel(const double* __restrict__ s, const double* __restrict__ in,
                       double* __restrict__ out, size_t n, size_t ld, int scale_half) {
  constexpr int TK = RB * NT, KC = mv::KC;
  // tw[i] = s_{d}, d = (TR ? row - inner : inner - row) over the chunk window;
  // hw[i] = s_{row + inner + p}. Threads read both at a stride of RB = 8
  // elements, so one pad slot per 8 (PX) keeps a warp's reads conflict free.
  constexpr int PADDED = TK + KC + (TK + KC) / 8;
  __shared__ double tw[PADDED];
  __shared__ double hw[PADDED];
  auto PX = [](int i) { return i + (i >> 3); };
  __shared__ double xv[KC];       // input at inner index (times pref for M^T)
  const int p = blockIdx.z;
  const size_t col = blockIdx.y;
  const size_t nr = (n + 1 - p) / 2;
  const size_t r0 = (size_t)blockIdx.x * TK;
  if (r0 >= nr) return;
  const double* x = in + col * ld;
  const int t = threadIdx.x;
  const size_t rt = r0 + (size_t)t * RB;  // this thread's first row
  double acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) acc[r] = 0.0;
  // inner range: forward b in [r0, nr); transpose a in [0, min(r0 + TK, nr))
  const size_t i_begin = TR ? 0 : r0;
  const size_t i_end = TR ? (r0 + TK < nr ? r0 + TK : nr) : nr;
  for (size_t i0 = i_begin; i0 < i_end; i0 += KC) {
    __syncthreads();
    // Toeplitz window: forward d = inner - row in [i0 - r0 - (TK-1), i0 - r0 + KC - 1]
    //                  transpose d = row - inner in [r0 - i0 - (KC-1), r0 - i0 + TK - 1]
    for (int q = t; q < TK + KC; q += NT) {
      const long long d = TR ? (long long)r0 - (long long)i0 - (KC - 1) + q
                             : (long long)i0 - (long long)r0 - (TK - 1) + q;
      tw[PX(q)] = (d >= 0 && d < (long long)n) ? s[d] : 0.0;
      const size_t h = r0 + i0 + p + q;  // row + inner + p, row - r0 + inner - i0 = q
      hw[PX(q)] = h < n ? s[h] : 0.0;
    }
    for (int q = t; q < KC; q += NT) {
      const size_t i = i0 + q;
      double v = 0.0;
      if (i < i_end && i < nr) {
        v = x[2 * i + p];
        if (TR && (2 * i + p) != 0) v *= 2.0;  // pref of row k = 2a + p of M
      }
      xv[q] = v;
    }
    __syncthreads();
    // Row r = rt + rr, inner i = i0 + j:
    //   forward   Toeplitz index (i - row) + (TK-1) - (i0 - r0) = j - (rt - r0) - rr + TK - 1
    //   transpose Toeplitz index (row - i) + (KC-1) - (r0 - i0) = (rt - r0) + rr - j + KC - 1
    //   Hankel index row + i - r0 - i0 = (rt - r0) + rr + j
    const int lr = (int)(rt - r0);
    double tv[RB], hv[RB];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      tv[rr] = TR ? tw[PX(lr + rr + KC - 1)] : tw[PX(TK - 1 - lr - rr)];
      hv[rr] = hw[PX(lr + rr)];
    }
    for (int j = 0; j < KC; j += RB) {
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int jj = j + u;  // tv/hv hold the factors of inner index i0 + jj
        const double xj = xv[jj];
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) acc[rr] = fma(tv[rr] * hv[rr], xj, acc[rr]);
        if (jj + 1 == KC) break;
        // slide: row rr at jj+1 takes row rr-1's Toeplitz factor at jj (both
        // directions) and row rr+1's Hankel factor; one new value each
#pragma unroll
        for (int rr = RB - 1; rr > 0; --rr) tv[rr] = tv[rr - 1];
        tv[0] = TR ? tw[PX(lr + KC - 2 - jj)] : tw[PX(TK - lr + jj)];
#pragma unroll
        for (int rr = 0; rr + 1 < RB; ++rr) hv[rr] = hv[rr + 1];
        hv[RB - 1] = hw[PX(lr + RB + jj)];
      }
    }
  }
  // write: forward pref (k == 0 ? 1 : 2); transpose optional (m + 1/2)
#pragma unroll
  for (int rr = 0; rr < RB; ++rr) {
    const size_t row = rt + rr;
    if (row >= nr) continue;
    const size_t k = 2 * row + p;
    double v = acc[rr];
    if (!TR)
      v *= (k == 0 ? 1.0 : 2.0);
    else if (scale_half)
      v *= (double)k + 0.5;
    out[col * ld + k] = v;
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
  if (cols <= 16 && n >= 2) {  // single vectors / few columns: tiled matrix-vector product
    if (n <= 8192) {
      constexpr int RB = 2, NT = 32;
      dim3 grid((unsigned)((rows + RB * NT - 1) / (RB * NT)), (unsigned)cols, 2);
      if (transpose)
        leg2cheb_mv_kernel<true, RB, NT><<<grid, NT, 0, st>>>(s, in, out, n, ld, scale_half);
      else
        leg2cheb_mv_kernel<false, RB, NT><<<grid, NT, 0, st>>>(s, in, out, n, ld, 0);
    } else {
      dim3 grid((unsigned)((rows + mv::TK - 1) / mv::TK), (unsigned)cols, 2);
      if (transpose)
        leg2cheb_mv_kernel<true><<<grid, mv::THREADS, 0, st>>>(s, in, out, n, ld, scale_half);
      else
        leg2cheb_mv_kernel<false><<<grid, mv::THREADS, 0, st>>>(s, in, out, n, ld, 0);
    }
    note_launch(transpose ? "leg2cheb_mv_kernel<T>" : "leg2cheb_mv_kernel<F>");
    return;
  }
  const bool aligned = (ld % 2 == 0) && (reinterpret_cast<uintptr_t>(in) % 16 == 0);
  if (aligned && n >= 64) {
    const size_t smem = mma::SMEM_DOUBLES * sizeof(double);
    for (size_t c0 = 0; c0 < cols; c0 += (size_t)65535 * mma::CT) {
      const size_t nc = cols - c0 < (size_t)65535 * mma::CT ? cols - c0 : (size_t)65535 * mma::CT;
      dim3 grid((unsigned)((rows + mma::RA - 1) / mma::RA), (unsigned)((nc + mma::CT - 1) / mma::CT));
      if (transpose) {
        FLB_CUDA(cudaFuncSetAttribute(leg2cheb_mma_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        leg2cheb_mma_kernel<true><<<grid, mma::THREADS, smem, st>>>(s, in + c0 * ld, out + c0 * ld,
                                                                    n, nc, ld, scale_half);
      } else {
        FLB_CUDA(cudaFuncSetAttribute(leg2cheb_mma_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        leg2cheb_mma_kernel<false><<<grid, mma::THREADS, smem, st>>>(s, in + c0 * ld, out + c0 * ld,
                                                                     n, nc, ld, 0);
      }
      note_launch(transpose ? "leg2cheb_mma_kernel<T>" : "leg2cheb_mma_kernel<F>");
    }
    return;
  }
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
