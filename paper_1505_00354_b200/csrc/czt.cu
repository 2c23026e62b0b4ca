// Generic DCT-III/DST-III engine and Taylor NDCT for any N and both grid
// kinds: a chirp-z (Bluestein) evaluation over power-of-two FFTs.
//
// Both grids are theta*_k = (k + kappa) 2 pi / D with
//   cheb1:    D = 2N,   kappa = 1/2   (trig.hpp:14-22, length-N REDFT01)
//   chebstar: D = 2N+1, kappa = 3/4   (odd slots of a length-(2N+1) REDFT01)
// so every operation of trig.hpp is a real or imaginary part of
//   forward:   Z_b = sum_a u_a e^{i a theta*_b}  (dct_iii = Re, dst_iii = Im)
//   transpose: Z_b = sum_a u_a e^{i b theta*_a}  (dct_iii_transpose = Re, ...)
// and e^{2 pi i ab/D} = e^{pi i a^2/D} e^{pi i b^2/D} e^{-pi i (b-a)^2/D}
// turns it into one linear convolution of length 2N-1 (FFT length P >= 2N-1).
// All chirp phases are reduced exactly in integers before one rounding.
//
// The Taylor NDCT (ndct.hpp:98-143) applies this L times with the n^l input
// scaling and delta^l/l! output weights fused into the load/store kernels,
// using the algebraically identical O(1)-magnitude split (n/N)^l (N delta)^l/l!
// (SURVEY.md 7 H9).
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "czt.cuh"
#include "fft.cuh"
#include "launch.cuh"

namespace flb {

namespace {

struct CztGeom {
  unsigned long long n;  // transform size N
  unsigned long long D;  // 2N (cheb1) or 2N+1 (chebstar)
  int kind;
  int log2p;
};

// e^{pi i (a^2 + 2 kappa a) / D}
__device__ __forceinline__ double2 chirp_kappa(const CztGeom& g, unsigned long long a) {
  if (g.kind == FL_CHEB1) return expi_pi_frac(a * a + a, g.D);
  return expi_pi_frac(2ull * a * a + 3ull * a, 2ull * g.D);
}
// e^{pi i a^2 / D}
__device__ __forceinline__ double2 chirp_plain(const CztGeom& g, unsigned long long a) {
  return expi_pi_frac(a * a, g.D);
}

// Per-element scale of the load/store side.
struct Scale {
  int mode;               // 0: 1, 1: (a/N)^l, 2: prod_{i<=l} (N delta_a / i)
  int l;
  double sign;            // taylor sign (store side)
  const double* delta;    // mode 2
  const double* mult;     // optional extra per-element factor (quadrature weights)
};

__device__ __forceinline__ double scale_of(const Scale& s, unsigned long long a, double nd) {
  double v = 1.0;
  if (s.mode == 1) {
    const double r = (double)a / nd;
    for (int i = 0; i < s.l; ++i) v *= r;
  } else if (s.mode == 2) {
    const double q = nd * s.delta[a];
    for (int i = 1; i <= s.l; ++i) v *= q / (double)i;
  }
  if (s.mult) v *= s.mult[a];
  return v;
}

__global__ void czt_load_kernel(CztGeom g, int transpose, int zero_first,
                                const double* __restrict__ in, size_t ld,
                                double2* __restrict__ A, Scale sc, int* nonfinite) {
  const unsigned long long P = 1ull << g.log2p;
  const size_t item = blockIdx.y;
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < P;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (t < g.n) {
      double x = in[item * ld + t] * scale_of(sc, t, (double)g.n);
      // term 0 carries scale 1 (or the IDLT weight): ndct.hpp:83-84 checks
      // exactly these values
      if (nonfinite && !isfinite(x)) atomicOr(nonfinite, 1);
      if (zero_first && t == 0) x = 0.0;
      const double2 ch = transpose ? chirp_plain(g, t) : chirp_kappa(g, t);
      v = make_double2(x * ch.x, x * ch.y);
    }
    A[item * P + t] = v;
  }
}

__global__ void czt_mul_kernel(double2* __restrict__ A, const double2* __restrict__ bhat,
                               int log2p, size_t total) {
  const unsigned long long mask = (1ull << log2p) - 1;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const double2 a = A[i], b = bhat[i & mask];
    A[i] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
}

// out[b] (+)= sign * scale(b) * (Re|Im)(chirp_out(b) * A[b])
__global__ void czt_store_kernel(CztGeom g, int transpose, int imag, int accumulate,
                                 int zero_first, const double2* __restrict__ A,
                                 double* __restrict__ out, size_t ld, Scale sc) {
  const unsigned long long P = 1ull << g.log2p;
  const size_t item = blockIdx.y;
  for (unsigned long long b = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; b < g.n;
       b += (unsigned long long)gridDim.x * blockDim.x) {
    const double2 ch = transpose ? chirp_kappa(g, b) : chirp_plain(g, b);
    const double2 z = cmul(A[item * P + b], ch);
    double v = imag ? z.y : z.x;
    if (zero_first && b == 0) v = 0.0;
    v = sc.sign * scale_of(sc, b, (double)g.n) * v;
    double* o = out + item * ld + b;
    *o = accumulate ? *o + v : v;
  }
}

__global__ void czt_kernel_fill(CztGeom g, double2* __restrict__ bvec) {
  const unsigned long long P = 1ull << g.log2p;
  const double invp = 1.0 / (double)P;  // exact: P is a power of two
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < P;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    unsigned long long m = 0;
    bool on = false;
    if (t < g.n) {
      m = t;
      on = true;
    } else if (t > P - g.n) {
      m = P - t;
      on = true;
    }
    if (on) {
      const double2 c = expi_pi_frac(m * m, g.D);
      v = make_double2(c.x * invp, -c.y * invp);  // e^{-pi i m^2 / D} / P
    }
    bvec[t] = v;
  }
}

struct CztPlan {
  CztGeom g;
  double2* bhat = nullptr;
};

const CztPlan& czt_plan(int kind, size_t n) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, size_t>, CztPlan> plans;
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  CztPlan& p = plans[{dev, kind, n}];
  if (!p.bhat) {
    CztGeom g;
    g.n = n;
    g.kind = kind;
    g.D = kind == FL_CHEB1 ? 2ull * n : 2ull * n + 1ull;
    int lg = 0;
    while ((1ull << lg) < 2ull * n - 1ull) ++lg;
    if (lg > kMaxLog2) fail(FL_RUNTIME_ERROR, "czt: transform size above the supported range");
    g.log2p = lg;
    const size_t P = 1ull << lg;
    double2 *b = nullptr, *scratch = nullptr;
    FLB_CUDA(cudaMalloc(&b, P * sizeof(double2)));
    if (lg > kMaxSmemLog2) FLB_CUDA(cudaMalloc(&scratch, P * sizeof(double2)));
    czt_kernel_fill<<<(unsigned)((P + 255) / 256 < 4096 ? (P + 255) / 256 : 4096), 256>>>(g, b);
    note_launch("czt_kernel_fill");
    fft_pow2(b, scratch, lg, 1, false, 0);
    FLB_CUDA(cudaDeviceSynchronize());
    if (scratch) FLB_CUDA(cudaFree(scratch));
    p.g = g;
    p.bhat = b;
  }
  return p;
}

unsigned grid_for(unsigned long long work, int threads) {
  unsigned long long g = (work + threads - 1) / threads;
  return (unsigned)(g < 1024 ? (g ? g : 1) : 1024);
}

// Runs one chirp-z term over `cols` columns.
void czt_term(const CztPlan& p, int transpose, int imag, const double* in, size_t ld_in,
              double* out, size_t ld_out, size_t cols, const Scale& load, const Scale& store,
              int accumulate, int* nonfinite, double2* A, double2* scratch, cudaStream_t s) {
  const unsigned long long P = 1ull << p.g.log2p;
  const int zero_first = imag ? 1 : 0;  // sin(0 * theta) = 0 exactly
  for (size_t c0 = 0; c0 < cols; c0 += 65535) {
    const size_t nc = cols - c0 < 65535 ? cols - c0 : 65535;
    dim3 grid(grid_for(P, 256), (unsigned)nc);
    czt_load_kernel<<<grid, 256, 0, s>>>(p.g, transpose, transpose ? 0 : zero_first,
                                         in + c0 * ld_in, ld_in, A + c0 * P, load, nonfinite);
    note_launch("czt_load_kernel");
  }
  fft_pow2(A, scratch, p.g.log2p, cols, false, s);
  czt_mul_kernel<<<grid_for(P * cols, 256) * 4, 256, 0, s>>>(A, p.bhat, p.g.log2p, P * cols);
  note_launch("czt_mul_kernel");
  fft_pow2(A, scratch, p.g.log2p, cols, true, s);
  for (size_t c0 = 0; c0 < cols; c0 += 65535) {
    const size_t nc = cols - c0 < 65535 ? cols - c0 : 65535;
    dim3 grid(grid_for(p.g.n, 256), (unsigned)nc);
    czt_store_kernel<<<grid, 256, 0, s>>>(p.g, transpose, imag, accumulate,
                                          transpose ? zero_first : 0, A + c0 * P,
                                          out + c0 * ld_out, ld_out, store);
    note_launch("czt_store_kernel");
  }
}

// Columns per chunk so that A (+ six-step scratch) stays within ~1 GiB.
size_t chunk_cols(const CztPlan& p, size_t batch) {
  const size_t P = 1ull << p.g.log2p;
  const size_t per = P * sizeof(double2) * (p.g.log2p > kMaxSmemLog2 ? 2 : 1);
  size_t c = (size_t(1) << 30) / per;
  if (c < 1) c = 1;
  return c < batch ? c : batch;
}

struct Scratch {
  double2* A = nullptr;
  double2* S = nullptr;
  cudaStream_t s;
  Scratch(const CztPlan& p, size_t cols, cudaStream_t st) : s(st) {
    const size_t P = 1ull << p.g.log2p;
    FLB_CUDA(cudaMallocAsync(&A, cols * P * sizeof(double2), s));
    if (p.g.log2p > kMaxSmemLog2) FLB_CUDA(cudaMallocAsync(&S, cols * P * sizeof(double2), s));
  }
  ~Scratch() {
    if (A) cudaFreeAsync(A, s);
    if (S) cudaFreeAsync(S, s);
  }
};

}  // namespace

void czt_trig(int op, int kind, size_t n, const double* in, double* out, size_t batch, size_t ld,
              cudaStream_t s) {
  const CztPlan& p = czt_plan(kind, n);
  const int transpose = op == FL_DCT_III_T || op == FL_DST_III_T;
  const int imag = op == FL_DST_III || op == FL_DST_III_T;
  const size_t chunk = chunk_cols(p, batch);
  Scratch sc(p, chunk, s);
  const Scale one{0, 0, 1.0, nullptr, nullptr};
  for (size_t c0 = 0; c0 < batch; c0 += chunk) {
    const size_t nc = batch - c0 < chunk ? batch - c0 : chunk;
    czt_term(p, transpose, imag, in + c0 * ld, ld, out + c0 * ld, ld, nc, one, one, 0, nullptr,
             sc.A, sc.S, s);
  }
}

static double taylor_sign(int l) { return ((l + 1) / 2) % 2 == 0 ? 1.0 : -1.0; }  // ndct.hpp:77

void czt_ndct(int transpose, int kind, size_t n, int num_terms, const double* delta,
              const double* in, double* out, size_t batch, size_t ld, const double* in_mult,
              int* nonfinite, cudaStream_t s, int l_lo, int l_hi) {
  if (l_hi < 0) l_hi = num_terms;
  const CztPlan& p = czt_plan(kind, n);
  const size_t chunk = chunk_cols(p, batch);
  Scratch sc(p, chunk, s);
  for (size_t c0 = 0; c0 < batch; c0 += chunk) {
    const size_t nc = batch - c0 < chunk ? batch - c0 : chunk;
    for (int l = l_lo; l < l_hi; ++l) {
      const int imag = l % 2;
      Scale load, store;
      if (!transpose) {
        // ndct.hpp:104-114: T_l((n/N)^l c) weighted by sign (N delta)^l / l!
        load = Scale{1, l, 1.0, nullptr, nullptr};
        store = Scale{2, l, taylor_sign(l), delta, nullptr};
      } else {
        // ndct.hpp:129-140: T_l^T((N delta)^l/l! g) weighted by sign (n/N)^l
        load = Scale{2, l, 1.0, delta, in_mult};
        store = Scale{1, l, taylor_sign(l), nullptr, nullptr};
      }
      czt_term(p, transpose, imag, in + c0 * ld, ld, out + c0 * ld, ld, nc, load, store, l > l_lo,
               l == 0 ? nonfinite : nullptr, sc.A, sc.S, s);
    }
  }
}

}  // namespace flb
