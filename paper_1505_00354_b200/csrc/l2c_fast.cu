// Fast Legendre <-> Chebyshev conversion for large N: Toeplitz-Hankel
// factorisation (the construction of Townsend, Webb & Olver, "Fast polynomial
// transforms based on Toeplitz and Hankel matrices", restated here).
//
// Per parity class p (rows k = 2a + p, inputs n = 2b + p) the reference's
// matrix (conversion.hpp:100-140) is the Hadamard product
//   A_{ab} = T_{ab} H_{ab},  T_{ab} = s_{b-a} [b >= a]  (upper Toeplitz),
//                            H_{ab} = s_{a+b+p}         (Hankel),
// with s_j = Lambda(j)/Lambda(0). H is a moment matrix of a positive measure
// (Lambda(z) = B(z+1/2, 1/2)/sqrt(pi)), hence positive definite and of low
// numerical rank: a pivoted Cholesky H ~ sum_{r<K} l_r l_r^T stopped at
// residual diagonal <= eps gives |A - sum_r D(l_r) T D(l_r)| <= eps
// entrywise, i.e. ||(A - A_K) x||_inf <= eps ||x||_1 (|s_j| <= 1). Then
//   A x   = sum_r l_r .* (T   (l_r .* x))   (T x: circular correlation),
//   A^T v = sum_r l_r .* (T^T (l_r .* v))   (T^T v: circular convolution),
// each a length-L >= 2 n_p FFT product with the fixed symbol FFT(s). Two rank
// terms ride in one complex FFT (real / imaginary parts: T is real). K grows
// like log N (measured 28 / 36 / 42 at N = 2^10 / 2^14 / 2^16), so the cost
// is O(K N log N) instead of the reference's N^2/4.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "l2c_fast.cuh"
#include "launch.cuh"

namespace flb {

struct L2CFast {
  size_t n = 0;
  int K[2] = {0, 0};
  size_t np[2] = {0, 0};
  int log2L[2] = {0, 0};
  double* ell[2] = {nullptr, nullptr};     // K x np, row r = l_r
  double2* shat[2] = {nullptr, nullptr};   // FFT_L of s~ (s_j for j < np);
                                           // th_symbol_layout order when L > 8192
};

namespace {

constexpr double kCholEps = 1e-17;  // residual diagonal bound (||A - A_K||_max)
constexpr int kMaxRank = 160;

// d_a = H_aa = s_{2a + p}
__global__ void chol_init_kernel(const double* __restrict__ s, int p, size_t np,
                                 double* __restrict__ d) {
  for (size_t a = blockIdx.x * (size_t)blockDim.x + threadIdx.x; a < np;
       a += (size_t)gridDim.x * blockDim.x)
    d[a] = s[2 * a + p];
}

// block-wise argmax of d (value, index)
__global__ void argmax_kernel(const double* __restrict__ d, size_t np, double* __restrict__ bv,
                              unsigned long long* __restrict__ bi) {
  __shared__ double sv[256];
  __shared__ unsigned long long si[256];
  double v = -1.0;
  unsigned long long idx = 0;
  for (size_t a = blockIdx.x * (size_t)blockDim.x + threadIdx.x; a < np;
       a += (size_t)gridDim.x * blockDim.x)
    if (d[a] > v) {
      v = d[a];
      idx = a;
    }
  sv[threadIdx.x] = v;
  si[threadIdx.x] = idx;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w && sv[threadIdx.x + w] > sv[threadIdx.x]) {
      sv[threadIdx.x] = sv[threadIdx.x + w];
      si[threadIdx.x] = si[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bv[blockIdx.x] = sv[0];
    bi[blockIdx.x] = si[0];
  }
}

// l_r(a) = (s_{a+i+p} - sum_{q<r} l_q(a) l_q(i)) / sqrt(d_i);  d_a -= l_r(a)^2
__global__ void chol_column_kernel(const double* __restrict__ s, int p, size_t np, size_t i,
                                   double di, double* __restrict__ ell, int r,
                                   const double* __restrict__ piv, double* __restrict__ d) {
  const double inv = 1.0 / sqrt(di);
  for (size_t a = blockIdx.x * (size_t)blockDim.x + threadIdx.x; a < np;
       a += (size_t)gridDim.x * blockDim.x) {
    double v = s[a + i + p];
    for (int q = 0; q < r; ++q) v -= ell[(size_t)q * np + a] * piv[q];
    v *= inv;
    ell[(size_t)r * np + a] = v;
    d[a] -= v * v;
  }
}

// piv[q] = l_q(i), q < r
__global__ void gather_pivot_kernel(const double* __restrict__ ell, size_t np, size_t i, int r,
                                    double* __restrict__ piv) {
  const int q = threadIdx.x + blockIdx.x * blockDim.x;
  if (q < r) piv[q] = ell[(size_t)q * np + i];
}

__global__ void symbol_kernel(const double* __restrict__ s, size_t np, size_t L,
                              double2* __restrict__ out) {
  for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < L;
       j += (size_t)gridDim.x * blockDim.x)
    out[j] = make_double2(j < np ? s[j] : 0.0, 0.0);
}

// V[q][b] = (l_{r0+2q}(b) u_b, l_{r0+2q+1}(b) u_b), u_b = x_{2b+p} (times the
// row prefactor of M for the transpose); zero for b >= np.
__global__ void th_pack_kernel(const double* __restrict__ x, int p, size_t n, size_t np,
                               size_t L, const double* __restrict__ ell, int K, int r0, int pairs,
                               int transpose, double2* __restrict__ V) {
  const int q = blockIdx.y;
  const int ra = r0 + 2 * q, rb = ra + 1;
  for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < L;
       b += (size_t)gridDim.x * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (b < np) {
      double u = x[2 * b + p];
      if (transpose && (2 * b + p) != 0) u *= 2.0;
      v.x = ell[(size_t)ra * np + b] * u;
      if (rb < K) v.y = ell[(size_t)rb * np + b] * u;
    }
    V[(size_t)q * L + b] = v;
  }
  (void)pairs;
  (void)n;
}

// V *= conj(S) (correlation, forward) or S (convolution, transpose)
__global__ void th_mul_kernel(double2* __restrict__ V, const double2* __restrict__ S, size_t L,
                              size_t total, int transpose) {
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const double2 a = V[t];
    double2 w = S[t % L];
    if (!transpose) w.y = -w.y;
    V[t] = make_double2(a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x);
  }
}

// y_a (+)= sum_q l_{r0+2q}(a) Re W_q[a] + l_{r0+2q+1}(a) Im W_q[a], scaled 1/L
__global__ void th_accum_kernel(const double2* __restrict__ W, size_t np, size_t L,
                                const double* __restrict__ ell, int K, int r0, int pairs,
                                double* __restrict__ y, int first) {
  const double inv = 1.0 / (double)L;  // exact: L is a power of two
  for (size_t a = blockIdx.x * (size_t)blockDim.x + threadIdx.x; a < np;
       a += (size_t)gridDim.x * blockDim.x) {
    double acc = first ? 0.0 : y[a];
    for (int q = 0; q < pairs; ++q) {
      const double2 w = W[(size_t)q * L + a];
      const int ra = r0 + 2 * q, rb = ra + 1;
      acc += ell[(size_t)ra * np + a] * (w.x * inv);
      if (rb < K) acc += ell[(size_t)rb * np + a] * (w.y * inv);
    }
    y[a] = acc;
  }
}

// out_{2a+p} = scale(2a+p) y_a
__global__ void th_store_kernel(const double* __restrict__ y, int p, size_t n, size_t np,
                                int transpose, int scale_half, double* __restrict__ out) {
  for (size_t a = blockIdx.x * (size_t)blockDim.x + threadIdx.x; a < np;
       a += (size_t)gridDim.x * blockDim.x) {
    const size_t k = 2 * a + p;
    if (k >= n) continue;
    double v = y[a];
    if (!transpose)
      v *= (k == 0 ? 1.0 : 2.0);
    else if (scale_half)
      v *= (double)k + 0.5;
    out[k] = v;
  }
}

unsigned grid1(size_t work) {
  const size_t g = (work + 255) / 256;
  return (unsigned)std::min<size_t>(g ? g : 1, (size_t)sm_count() * 16);
}

}  // namespace

L2CFast* l2c_fast_create(size_t n, const double* s, cudaStream_t st) {
  if (n < 4) return nullptr;
  L2CFast* f = new L2CFast;
  f->n = n;
  try {
    for (int p = 0; p < 2; ++p) {
      const size_t np = (n + 1 - p) / 2;
      f->np[p] = np;
      int lg = 0;
      while ((size_t(1) << lg) < 2 * np) ++lg;
      f->log2L[p] = lg;
      if (lg > kMaxLog2) fail(FL_RUNTIME_ERROR, "leg2cheb fast: size above the supported range");
      // pivoted Cholesky of H (device), rank grows as needed
      double *d = nullptr, *piv = nullptr, *bv = nullptr;
      unsigned long long* bi = nullptr;
      const unsigned gb = grid1(np);
      FLB_CUDA(cudaMallocAsync(&d, np * sizeof(double), st));
      FLB_CUDA(cudaMallocAsync(&piv, kMaxRank * sizeof(double), st));
      FLB_CUDA(cudaMallocAsync(&bv, gb * sizeof(double), st));
      FLB_CUDA(cudaMallocAsync(&bi, gb * sizeof(unsigned long long), st));
      // capacity from the observed growth (~2.3 per doubling of N), grown on demand
      int lgn = 0;
      while ((size_t(1) << lgn) < np) ++lgn;
      int cap = std::min(kMaxRank, 24 + 3 * lgn);
      FLB_CUDA(cudaMalloc(&f->ell[p], (size_t)cap * np * sizeof(double)));
      chol_init_kernel<<<gb, 256, 0, st>>>(s, p, np, d);
      note_launch("chol_init_kernel");
      std::vector<double> hv(gb);
      std::vector<unsigned long long> hi(gb);
      int r = 0;
      for (; r < kMaxRank; ++r) {
        if (r == cap) {
          const int ncap = std::min(kMaxRank, cap + cap / 2);
          double* grown = nullptr;
          FLB_CUDA(cudaMalloc(&grown, (size_t)ncap * np * sizeof(double)));
          FLB_CUDA(cudaMemcpyAsync(grown, f->ell[p], (size_t)cap * np * sizeof(double),
                                   cudaMemcpyDeviceToDevice, st));
          FLB_CUDA(cudaStreamSynchronize(st));
          cudaFree(f->ell[p]);
          f->ell[p] = grown;
          cap = ncap;
        }
        argmax_kernel<<<gb, 256, 0, st>>>(d, np, bv, bi);
        note_launch("argmax_kernel");
        FLB_CUDA(cudaMemcpyAsync(hv.data(), bv, gb * sizeof(double), cudaMemcpyDeviceToHost, st));
        FLB_CUDA(cudaMemcpyAsync(hi.data(), bi, gb * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, st));
        FLB_CUDA(cudaStreamSynchronize(st));
        size_t best = 0;
        for (unsigned b = 1; b < gb; ++b)
          if (hv[b] > hv[best]) best = b;
        const double di = hv[best];
        const size_t i = hi[best];
        if (!(di > kCholEps)) break;
        if (r > 0) {
          gather_pivot_kernel<<<(r + 127) / 128, 128, 0, st>>>(f->ell[p], np, i, r, piv);
          note_launch("gather_pivot_kernel");
        }
        chol_column_kernel<<<gb, 256, 0, st>>>(s, p, np, i, di, f->ell[p], r, piv, d);
        note_launch("chol_column_kernel");
      }
      if (r == kMaxRank) fail(FL_RUNTIME_ERROR, "leg2cheb fast: Hankel rank above the cap");
      f->K[p] = r;
      cudaFreeAsync(d, st);
      cudaFreeAsync(piv, st);
      cudaFreeAsync(bv, st);
      cudaFreeAsync(bi, st);
      // symbol FFT
      const size_t L = size_t(1) << lg;
      FLB_CUDA(cudaMalloc(&f->shat[p], L * sizeof(double2)));
      double2* scratch = nullptr;
      if (lg > kMaxSmemLog2) FLB_CUDA(cudaMallocAsync(&scratch, L * sizeof(double2), st));
      symbol_kernel<<<grid1(L), 256, 0, st>>>(s, np, L, f->shat[p]);
      note_launch("symbol_kernel");
      fft_pow2(f->shat[p], scratch, lg, 1, false, st);
      // the fused sweep reads the spectrum in its row-pass order
      if (lg > kMaxSmemLog2) th_symbol_layout(f->shat[p], scratch, lg, st);
      if (scratch) cudaFreeAsync(scratch, st);
    }
    FLB_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    l2c_fast_destroy(f);
    throw;
  }
  return f;
}

void l2c_fast_destroy(L2CFast* f) {
  if (!f) return;
  for (int p = 0; p < 2; ++p) {
    if (f->ell[p]) cudaFree(f->ell[p]);
    if (f->shat[p]) cudaFree(f->shat[p]);
  }
  delete f;
}

int l2c_fast_rank(const L2CFast& f, int parity) { return f.K[parity]; }

void l2c_fast_apply(const L2CFast& f, int transpose, const double* in, double* out, size_t cols,
                    size_t ld, int scale_half, cudaStream_t st, int r_lo, int r_hi) {
  const size_t n = f.n;
  for (int p = 0; p < 2; ++p) {
    const size_t np = f.np[p];
    if (np == 0) continue;
    const int lg = f.log2L[p];
    const size_t L = size_t(1) << lg;
    // rank terms [r_lo, r_hi) of this parity (a partial sum for the
    // rank-parallel multi-GPU path; all of them by default)
    const int K = r_hi < 0 ? f.K[p] : std::min(r_hi, f.K[p]);
    const int r_first = std::min(std::max(r_lo, 0), K);
    const int pairs_total = (K - r_first + 1) / 2;
    // rank pairs per batched FFT, bounded to ~2 GiB of work buffers
    const size_t cap = std::max<size_t>(1, (size_t(1) << 31) / (2 * L * sizeof(double2)));
    const int chunk = (int)std::max<size_t>(1, std::min<size_t>(cap, (size_t)pairs_total));
    double2 *V = nullptr, *S = nullptr;
    double* y = nullptr;
    FLB_CUDA(cudaMallocAsync(&V, (size_t)chunk * L * sizeof(double2), st));
    if (lg > kMaxSmemLog2) FLB_CUDA(cudaMallocAsync(&S, (size_t)chunk * L * sizeof(double2), st));
    FLB_CUDA(cudaMallocAsync(&y, np * sizeof(double), st));
    for (size_t c = 0; c < cols; ++c) {
      const double* x = in + c * ld;
      if (pairs_total == 0) FLB_CUDA(cudaMemsetAsync(y, 0, np * sizeof(double), st));
      for (int q0 = 0; q0 < pairs_total; q0 += chunk) {
        const int pq = std::min(chunk, pairs_total - q0);
        if (lg > kMaxSmemLog2) {
          // packing and symbol product inside the FFT passes
          const ThArgs a{x, p, np, f.ell[p], K, r_first + 2 * q0, transpose, f.shat[p]};
          th_sweep(a, lg, (size_t)pq, V, S, st);
          th_accum_kernel<<<grid1(np), 256, 0, st>>>(V, np, L, f.ell[p], K, r_first + 2 * q0, pq,
                                                      y, q0 == 0);
          note_launch("th_accum_kernel");
          continue;
        }
        dim3 g(grid1(L), (unsigned)pq);
        th_pack_kernel<<<g, 256, 0, st>>>(x, p, n, np, L, f.ell[p], K, r_first + 2 * q0, pq,
                                           transpose, V);
        note_launch("th_pack_kernel");
        fft_pow2(V, S, lg, pq, false, st);
        th_mul_kernel<<<grid1((size_t)pq * L), 256, 0, st>>>(V, f.shat[p], L, (size_t)pq * L,
                                                              transpose);
        note_launch("th_mul_kernel");
        fft_pow2(V, S, lg, pq, true, st);
        th_accum_kernel<<<grid1(np), 256, 0, st>>>(V, np, L, f.ell[p], K, r_first + 2 * q0, pq,
                                                    y, q0 == 0);
        note_launch("th_accum_kernel");
      }
      th_store_kernel<<<grid1(np), 256, 0, st>>>(y, p, n, np, transpose, scale_half,
                                                  out + c * ld);
      note_launch("th_store_kernel");
    }
    cudaFreeAsync(V, st);
    if (S) cudaFreeAsync(S, st);
    cudaFreeAsync(y, st);
  }
}

}  // namespace flb
