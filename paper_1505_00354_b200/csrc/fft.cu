// Batched power-of-two complex fp64 FFT: shared-memory Stockham for
// P <= 8192, six-step (transpose / row FFTs / twiddle-transpose / row FFTs /
// transpose) through HBM above that.
#include <map>
#include <mutex>
#include <cmath>
#include <utility>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "launch.cuh"

namespace flb {

namespace {

__global__ void twiddle_kernel(double2* tw, unsigned long long p) {
  const unsigned long long m = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (m >= p) return;
  double s, c;
  sincospi(2.0 * (double)m / (double)p, &s, &c);
  tw[m] = make_double2(c, -s);
}

template <int LOG2P, bool INV>
__global__ void __launch_bounds__(512) fft_smem_kernel(double2* __restrict__ data, size_t rows,
                                                       const double2* __restrict__ tw) {
  constexpr int P = 1 << LOG2P;
  constexpr int E = P >= 8192 ? 16 : 8;
  constexpr int TR = P / E;
  constexpr int RPC = TR >= 256 ? 1 : 256 / TR;
  extern __shared__ double2 sm[];
  const size_t row0 = (size_t)blockIdx.x * RPC;
  for (int i = threadIdx.x; i < RPC * P; i += blockDim.x) {
    const size_t r = row0 + i / P;
    sm[(i / P) * smem_row(P) + smem_pad(i % P)] = r < rows ? data[r * P + (i % P)] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int lr = threadIdx.x / TR, tid = threadIdx.x % TR;
  fft_row_smem<P, E, INV>(sm + lr * smem_row(P), tid, tw);
  for (int i = threadIdx.x; i < RPC * P; i += blockDim.x) {
    const size_t r = row0 + i / P;
    if (r < rows) data[r * P + (i % P)] = sm[(i / P) * smem_row(P) + smem_pad(i % P)];
  }
}

// P in {1, 2, 4}: direct DFT, one thread per row
template <bool INV>
__global__ void fft_tiny_kernel(double2* __restrict__ data, size_t rows, int p) {
  const size_t r = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double2 v[4], o[4];
  for (int i = 0; i < p; ++i) v[i] = data[r * p + i];
  for (int k = 0; k < p; ++k) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < p; ++j) {
      const int m = (j * k) % p;
      double s, c;
      sincospi(2.0 * (double)m / (double)p, &s, &c);
      if (!INV) s = -s;
      acc.x += v[j].x * c - v[j].y * s;
      acc.y += v[j].x * s + v[j].y * c;
    }
    o[k] = acc;
  }
  for (int i = 0; i < p; ++i) data[r * p + i] = o[i];
}

// out[item][c][r] = in[item][r][c] * (twiddle ? w_P^{r c} : 1)
template <bool INV>
__global__ void transpose_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                 int rows, int cols, unsigned long long twiddle_p) {
  __shared__ double2 tile[32][33];
  const size_t item = blockIdx.z;
  const size_t plane = (size_t)rows * cols;
  const double2* src = in + item * plane;
  double2* dst = out + item * plane;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    const int r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = src[(size_t)r * cols + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    const int c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) {
      double2 v = tile[threadIdx.x][dy];
      if (twiddle_p) {
        const unsigned long long m = ((unsigned long long)r * (unsigned long long)c) % twiddle_p;
        double s, co;
        sincospi(2.0 * (double)m / (double)twiddle_p, &s, &co);
        if (!INV) s = -s;
        v = make_double2(v.x * co - v.y * s, v.x * s + v.y * co);
      }
      dst[(size_t)c * rows + r] = v;
    }
  }
}

// ---- multi-pass FFT for P > 8192 ---------------------------------------------
// P = R C: x[a1 + R a2] -> X[b2 + C b1]. The length-C transform over a2 (per
// a1) is one line pass (C <= 4096) or two (C = C1 C2, a2 = c1 + C1 c2); the
// twiddle w_P^{a1 b2} is applied on its way out, and a last pass transforms
// the contiguous rows over a1 and writes X transposed. Every pass is a "line"
// FFT in shared memory over lines of length L <= 4096: line l (lo = l mod M,
// hi = l / M) reads src[lo + hi Hin + e Sin] and writes
// dst[lo + hi Hout + k Sout] * w_Q^{lo (hi u + k v) + hi k z}. CTAs take
// adjacent lines (adjacent lo), so every global access is a run of
// LINES * 16 B. Six-step needed six read+write passes; this needs two (P <=
// 2^23) or three.
struct LineMap {
  unsigned long long M, Hin, Sin, Hout, Sout;   // addressing (M a power of two)
  unsigned long long Q, u, v, z;                // twiddle exponent (Q = 0: none; a power of two)
};

template <int LOG2L>
struct LinePass {
  static constexpr int L = 1 << LOG2L;
  static constexpr int E = 8;
  static constexpr int TL = L / E;                                   // threads per line
  static constexpr int LINES = L >= 4096 ? 2 : L >= 1024 ? 4 : 8;    // lines per CTA
  static constexpr int THREADS = TL * LINES;
  // per-line named barriers need whole warps; short lines sync CTA-wide
  static constexpr int GT = TL % 32 != 0 ? 0 : TL;
  // line stride in smem: one extra element so the LINES lines that a warp's
  // global-order loads / stores touch fall in different banks
  static constexpr int LS = smem_row(L) + 1;
  static constexpr size_t SMEM = (size_t)LINES * LS * sizeof(double2);
};

template <int LOG2L, bool INV>
__global__ void __launch_bounds__(LinePass<LOG2L>::THREADS)
    fft_line_kernel(const double2* __restrict__ src, double2* __restrict__ dst,
                    unsigned long long P, LineMap mp, const double2* __restrict__ tw) {
  using Q = LinePass<LOG2L>;
  constexpr int L = Q::L, LINES = Q::LINES;
  extern __shared__ double2 sm[];
  const size_t item = blockIdx.y;
  const double2* x = src + item * P;
  double2* y = dst + item * P;
  const unsigned long long l0 = (unsigned long long)blockIdx.x * LINES;
  const unsigned long long mmask = mp.M - 1, qmask = mp.Q - 1;
  const int mshift = __ffsll((long long)mp.M) - 1;
  const bool rows_in = mp.Sin == 1;  // contiguous lines: element index fastest
  for (int i = threadIdx.x; i < LINES * L; i += blockDim.x) {
    const int j = rows_in ? i / L : i % LINES, e = rows_in ? i % L : i / LINES;
    const unsigned long long l = l0 + j, lo = l & mmask, hi = l >> mshift;
    sm[j * Q::LS + smem_pad(e)] = x[lo + hi * mp.Hin + (unsigned long long)e * mp.Sin];
  }
  __syncthreads();
  const int line = threadIdx.x / Q::TL, tid = threadIdx.x % Q::TL;
  fft_row_smem<L, Q::E, INV, Q::GT>(sm + line * Q::LS, tid, tw, 1 + line);
  __syncthreads();
  for (int i = threadIdx.x; i < LINES * L; i += blockDim.x) {
    const int j = i % LINES, k = i / LINES;
    const unsigned long long l = l0 + j, lo = l & mmask, hi = l >> mshift;
    double2 v = sm[j * Q::LS + smem_pad(k)];
    if (mp.Q) {
      const unsigned long long kk = (unsigned long long)k;
      // exponent mod Q by masks (wrap-around of the 64-bit products is harmless mod 2^k)
      const unsigned long long m = (lo * (hi * mp.u + kk * mp.v) + hi * kk * mp.z) & qmask;
      double sn, cs;
      sincospi(2.0 * (double)m / (double)mp.Q, &sn, &cs);
      if (!INV) sn = -sn;
      v = make_double2(v.x * cs - v.y * sn, v.x * sn + v.y * cs);
    }
    y[lo + hi * mp.Hout + (unsigned long long)k * mp.Sout] = v;
  }
}

template <int LOG2L, bool INV>
void launch_line(const double2* src, double2* dst, unsigned long long P, size_t items,
                 const LineMap& mp, cudaStream_t s) {
  using Q = LinePass<LOG2L>;
  const double2* tw = pass_twiddles(LOG2L);
  const unsigned long long lines = P >> LOG2L;
  FLB_CUDA(cudaFuncSetAttribute(fft_line_kernel<LOG2L, INV>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM));
  dim3 grid((unsigned)(lines / Q::LINES), (unsigned)items);
  fft_line_kernel<LOG2L, INV><<<grid, Q::THREADS, Q::SMEM, s>>>(src, dst, P, mp, tw);
  note_launch("fft_line_kernel");
}

template <bool INV>
void line_pass(int log2l, const double2* src, double2* dst, unsigned long long P, size_t items,
               const LineMap& mp, cudaStream_t s) {
  switch (log2l) {
    case 5: launch_line<5, INV>(src, dst, P, items, mp, s); break;
    case 6: launch_line<6, INV>(src, dst, P, items, mp, s); break;
    case 7: launch_line<7, INV>(src, dst, P, items, mp, s); break;
    case 8: launch_line<8, INV>(src, dst, P, items, mp, s); break;
    case 9: launch_line<9, INV>(src, dst, P, items, mp, s); break;
    case 10: launch_line<10, INV>(src, dst, P, items, mp, s); break;
    case 11: launch_line<11, INV>(src, dst, P, items, mp, s); break;
    case 12: launch_line<12, INV>(src, dst, P, items, mp, s); break;
    default: fail(FL_RUNTIME_ERROR, "fft: unsupported line length");
  }
}

template <bool INV>
void fft_multipass(double2* d, double2* t, int log2p, size_t items, cudaStream_t s) {
  const unsigned long long P = 1ull << log2p;
  const int passes = log2p <= 24 ? 2 : 3;
  const int lr = passes == 2 ? log2p / 2 : log2p / 3;  // rows (last pass)
  const int lc = log2p - lr;
  const unsigned long long R = 1ull << lr, C = 1ull << lc;
  if (passes == 2) {
    // columns over a2 (stride R), twiddle w_P^{a1 b2}: d -> t at a1 + R b2
    line_pass<INV>(lc, d, t, P, items, LineMap{R, 0, R, 0, R, P, 0, 1, 0}, s);
  } else {
    const int l1 = lc / 2, l2 = lc - l1;  // a2 = c1 + C1 c2
    const unsigned long long C1 = 1ull << l1, C2 = 1ull << l2;
    // over c2 (stride R C1), in place, twiddle w_C^{c1 d2}: lines l = a1 + R c1
    line_pass<INV>(l2, d, d, P, items, LineMap{R, R, R * C1, R, R * C1, C, 0, 0, 1}, s);
    // over c1 (stride R) -> t at a1 + R (d2 + C2 d1), twiddle w_P^{a1 (d2 + C2 d1)};
    // lines l = a1 + R d2: lo = a1, hi = d2
    line_pass<INV>(l1, d, t, P, items, LineMap{R, R * C1, R, R, R * C2, P, 1, C2, 0}, s);
  }
  // rows over a1 (contiguous), written transposed to X[b2 + C b1]: lines l = b2
  line_pass<INV>(lr, t, d, P, items, LineMap{1, R, 1, 1, C, 0, 0, 0, 0}, s);
}

template <int LOG2P, bool INV>
void launch_smem(double2* data, size_t rows, const double2* tw, cudaStream_t s) {
  constexpr int P = 1 << LOG2P;
  constexpr int E = P >= 8192 ? 16 : 8;
  constexpr int TR = P / E;
  constexpr int RPC = TR >= 256 ? 1 : 256 / TR;
  const size_t smem = (size_t)RPC * smem_row(P) * sizeof(double2);
  FLB_CUDA(cudaFuncSetAttribute(fft_smem_kernel<LOG2P, INV>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const size_t grid = (rows + RPC - 1) / RPC;
  fft_smem_kernel<LOG2P, INV><<<(unsigned)grid, TR * RPC, smem, s>>>(data, rows, tw);
  note_launch("fft_smem_kernel");
}

template <bool INV>
void launch_smem_dispatch(int log2p, double2* data, size_t rows, const double2* tw,
                          cudaStream_t s) {
  switch (log2p) {
    case 3: launch_smem<3, INV>(data, rows, tw, s); break;
    case 4: launch_smem<4, INV>(data, rows, tw, s); break;
    case 5: launch_smem<5, INV>(data, rows, tw, s); break;
    case 6: launch_smem<6, INV>(data, rows, tw, s); break;
    case 7: launch_smem<7, INV>(data, rows, tw, s); break;
    case 8: launch_smem<8, INV>(data, rows, tw, s); break;
    case 9: launch_smem<9, INV>(data, rows, tw, s); break;
    case 10: launch_smem<10, INV>(data, rows, tw, s); break;
    case 11: launch_smem<11, INV>(data, rows, tw, s); break;
    case 12: launch_smem<12, INV>(data, rows, tw, s); break;
    case 13: launch_smem<13, INV>(data, rows, tw, s); break;
    default: fail(FL_RUNTIME_ERROR, "fft: unsupported shared-memory size");
  }
}

void transpose(const double2* in, double2* out, int rows, int cols, size_t items,
               unsigned long long twiddle_p, bool inverse, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, (unsigned)items);
  if (items > 65535) fail(FL_RUNTIME_ERROR, "fft: too many transforms in one six-step call");
  if (inverse)
    transpose_kernel<true><<<grid, block, 0, s>>>(in, out, rows, cols, twiddle_p);
  else
    transpose_kernel<false><<<grid, block, 0, s>>>(in, out, rows, cols, twiddle_p);
  note_launch("transpose_kernel");
}

void fft_rows(double2* data, int log2p, size_t rows, bool inverse, cudaStream_t s) {
  if (log2p <= 2) {
    const int threads = 128;
    const unsigned grid = (unsigned)((rows + threads - 1) / threads);
    if (inverse)
      fft_tiny_kernel<true><<<grid, threads, 0, s>>>(data, rows, 1 << log2p);
    else
      fft_tiny_kernel<false><<<grid, threads, 0, s>>>(data, rows, 1 << log2p);
    note_launch("fft_tiny_kernel");
    return;
  }
  const double2* tw = pass_twiddles(log2p);
  if (inverse)
    launch_smem_dispatch<true>(log2p, data, rows, tw, s);
  else
    launch_smem_dispatch<false>(log2p, data, rows, tw, s);
}

}  // namespace

const double2* twiddle_table(int log2p) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, double2*> tables;
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  double2*& slot = tables[{dev, log2p}];
  if (!slot) {
    const unsigned long long p = 1ull << log2p;
    FLB_CUDA(cudaMalloc(&slot, p * sizeof(double2)));
    twiddle_kernel<<<(unsigned)((p + 255) / 256), 256>>>(slot, p);
    note_launch("twiddle_kernel");
    FLB_CUDA(cudaDeviceSynchronize());
  }
  return slot;
}

const double2* pass_twiddles(int log2p) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, double2*> tables;
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  double2*& slot = tables[{dev, log2p}];
  if (!slot) {
    const int p = 1 << log2p;
    std::vector<double2> h;
    h.reserve(twiddle_entries(p) + 1);
    const long double pi_l = 3.14159265358979323846264338327950288L;
    for (int ns = 1; ns < p; ns *= pass_radix(p, ns)) {
      const int r_ = pass_radix(p, ns);
      if (ns == 1) continue;
      for (int r = 1; r < r_; ++r)
        for (int k = 0; k < ns; ++k) {
          // w_{ns R}^{r k} = e^{-2 pi i r k / (ns R)}, phase reduced exactly
          const long long m = (long long)r * k % (long long)(ns * r_);
          const long double a = 2.0L * pi_l * (long double)m / (long double)(ns * r_);
          h.push_back(make_double2((double)cosl(a), (double)-sinl(a)));
        }
    }
    if (h.empty()) h.push_back(make_double2(1.0, 0.0));
    FLB_CUDA(cudaMalloc(&slot, h.size() * sizeof(double2)));
    FLB_CUDA(cudaMemcpy(slot, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  }
  return slot;
}

void fft_pow2(double2* data, double2* scratch, int log2p, size_t batch, bool inverse,
              cudaStream_t s) {
  if (log2p < 0 || log2p > kMaxLog2) fail(FL_RUNTIME_ERROR, "fft: length out of range");
  if (batch == 0) return;
  if (log2p <= kMaxSmemLog2) {
    fft_rows(data, log2p, batch, inverse, s);
    return;
  }
  const unsigned long long P = 1ull << log2p;
  for (size_t b0 = 0; b0 < batch; b0 += 65535) {
    const size_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    if (inverse)
      fft_multipass<true>(data + b0 * P, scratch + b0 * P, log2p, nb, s);
    else
      fft_multipass<false>(data + b0 * P, scratch + b0 * P, log2p, nb, s);
  }
}

}  // namespace flb
