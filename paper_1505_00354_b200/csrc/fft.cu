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
  // two-level twiddle tables of w_Q (filled by launch_line when Q != 0):
  // w_Q^m = twlo[m mod 2^twh] * twhi[m >> twh]
  const double2* twlo = nullptr;
  const double2* twhi = nullptr;
  int twh = 0;
};

// w_Q^j = e^{-2 pi i j/Q} for j < 2^h (lo) and j = 2^h i, i < Q / 2^h (hi),
// h = ceil(log2 Q / 2): one complex product per twiddle instead of an fp64
// sincospi (the twiddled line passes were issue-bound on it: 1.6x the time
// of the untwiddled pass at 2^26). Phases reduced exactly, long double.
std::pair<const double2*, const double2*> twiddle_pair(int log2q) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, std::pair<double2*, double2*>> tables;
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = tables[{dev, log2q}];
  if (!slot.first) {
    const int h = (log2q + 1) / 2;
    const long long q = 1ll << log2q, nlo = 1ll << h, nhi = q >> h;
    const long double pi_l = 3.14159265358979323846264338327950288L;
    std::vector<double2> lo(nlo), hi(nhi);
    for (long long j = 0; j < nlo; ++j) {
      const long double a = 2.0L * pi_l * (long double)j / (long double)q;
      lo[j] = make_double2((double)cosl(a), (double)-sinl(a));
    }
    for (long long i = 0; i < nhi; ++i) {
      const long double a = 2.0L * pi_l * (long double)(i * nlo) / (long double)q;
      hi[i] = make_double2((double)cosl(a), (double)-sinl(a));
    }
    FLB_CUDA(cudaMalloc(&slot.first, nlo * sizeof(double2)));
    FLB_CUDA(cudaMalloc(&slot.second, nhi * sizeof(double2)));
    FLB_CUDA(cudaMemcpy(slot.first, lo.data(), nlo * sizeof(double2), cudaMemcpyHostToDevice));
    FLB_CUDA(cudaMemcpy(slot.second, hi.data(), nhi * sizeof(double2), cudaMemcpyHostToDevice));
  }
  return {slot.first, slot.second};
}

// lines per CTA of a pass over lines of 2^log2l
constexpr int line_ctas_lines(int log2l) { return log2l >= 12 ? 2 : log2l >= 10 ? 4 : 8; }

template <int LOG2L>
struct LinePass {
  static constexpr int L = 1 << LOG2L;
  static constexpr int E = 8;
  static constexpr int TL = L / E;                                   // threads per line
  static constexpr int LINES = line_ctas_lines(LOG2L);
  static constexpr int THREADS = TL * LINES;
  // per-line named barriers need whole warps; short lines sync CTA-wide
  static constexpr int GT = TL % 32 != 0 ? 0 : TL;
  // line stride in smem: one extra element so the LINES lines that a warp's
  // global-order loads / stores touch fall in different banks
  static constexpr int LS = smem_row(L) + 1;
  static constexpr size_t SMEM = (size_t)LINES * LS * sizeof(double2);
};

// What a line pass reads (IN: IO_PACK builds the Toeplitz-Hankel operand from
// x and the l_r rows) and whether it is the fused row pass (MID: forward
// transform, symbol product, inverse transform).
enum { IO_PLAIN = 0, IO_PACK = 1 };
// Loads of a pass issued all at once (registers) before the shared-memory
// stores: faster for lines of <= 512 points (2^26: 327 vs 338 ms per C5
// DLT), slower above (2^20: 4.11 vs 3.78 ms per C3 DLT).
constexpr bool line_unroll(int log2l) { return log2l <= 9; }
struct LineIO {
  const double2* src;
  double2* dst;
  ThArgs th;
};

__device__ __forceinline__ double2 th_pack_value(const ThArgs& a, size_t item,
                                                 unsigned long long b) {
  double2 v = make_double2(0.0, 0.0);
  if (b < a.np) {
    const unsigned long long k = 2 * b + a.p;
    double u = a.x[k];
    if (a.transpose && k != 0) u *= 2.0;
    const int ra = a.ra0 + 2 * (int)item;
    v.x = a.ell[(size_t)ra * a.np + b] * u;
    if (ra + 1 < a.K) v.y = a.ell[(size_t)(ra + 1) * a.np + b] * u;
  }
  return v;
}

template <int LOG2L, bool INV, int IN, bool MID>
__global__ void __launch_bounds__(LinePass<LOG2L>::THREADS)
    fft_line_kernel(LineIO io, unsigned long long P, LineMap mp, const double2* __restrict__ tw) {
  using Q = LinePass<LOG2L>;
  constexpr int L = Q::L, LINES = Q::LINES, PER = LINES * L / Q::THREADS;
  // the store twiddle belongs to the direction of the last transform
  constexpr bool TW_INV = MID ? !INV : INV;
  extern __shared__ double2 sm[];
  // element indices within one item are < P <= 2^27: 32-bit arithmetic (the
  // 64-bit index products were a large share of the pass's issue slots);
  // twiddle exponents mod Q | 2^32 are exact in wrapping 32-bit products
  const uint32_t l0 = blockIdx.x * (uint32_t)LINES;
  const uint32_t mmask = (uint32_t)mp.M - 1u, qmask = (uint32_t)(mp.Q - 1);
  const int mshift = __ffsll((long long)mp.M) - 1;
  const uint32_t Hin = (uint32_t)mp.Hin, Sin = (uint32_t)mp.Sin, Hout = (uint32_t)mp.Hout,
                 Sout = (uint32_t)mp.Sout;
  const uint32_t tu = (uint32_t)mp.u, tv = (uint32_t)mp.v, tz = (uint32_t)mp.z;
  const bool rows_in = mp.Sin == 1;   // contiguous lines: element index fastest
  const bool rows_out = mp.Sout == 1;
  const int line = threadIdx.x / Q::TL, tid = threadIdx.x % Q::TL;
  // MID: the symbol rows of this CTA's lines, staged next to the data when
  // both fit (else read in the product loop)
  constexpr bool SYM_SMEM = MID && 2 * Q::SMEM <= 80 * 1024;  // keeps >= 2 CTAs per SM
  double2* sym_s = sm + LINES * Q::LS;
  {
    const size_t item = blockIdx.y;
    const double2* src_item = IN == IO_PACK ? nullptr : io.src + item * P;
    double2* dst_item = io.dst + item * P;
    // all PER loads of a thread are issued before the first smem store
    if constexpr (line_unroll(LOG2L)) {
      double2 v[PER];
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int i = threadIdx.x + r * Q::THREADS;
        const int j = rows_in ? i / L : i % LINES, e = rows_in ? i % L : i / LINES;
        const uint32_t l = l0 + j, lo = l & mmask, hi = l >> mshift;
        const uint32_t g = lo + hi * Hin + (uint32_t)e * Sin;
        if constexpr (IN == IO_PACK)
          v[r] = th_pack_value(io.th, item, g);
        else
          v[r] = src_item[g];
      }
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int i = threadIdx.x + r * Q::THREADS;
        const int j = rows_in ? i / L : i % LINES, e = rows_in ? i % L : i / LINES;
        sm[j * Q::LS + smem_pad(e)] = v[r];
      }
    } else {
      for (int i = threadIdx.x; i < LINES * L; i += blockDim.x) {
        const int j = rows_in ? i / L : i % LINES, e = rows_in ? i % L : i / LINES;
        const uint32_t l = l0 + j, lo = l & mmask, hi = l >> mshift;
        const uint32_t g = lo + hi * Hin + (uint32_t)e * Sin;
        double2 v;
        if constexpr (IN == IO_PACK)
          v = th_pack_value(io.th, item, g);
        else
          v = src_item[g];
        sm[j * Q::LS + smem_pad(e)] = v;
      }
    }
    if constexpr (SYM_SMEM) {
      for (int i = threadIdx.x; i < LINES * L; i += blockDim.x) {
        double2 w = io.th.sym[(l0 + i / L) * L + i % L];
        if (!io.th.transpose) w.y = -w.y;
        sym_s[(i / L) * Q::LS + smem_pad(i % L)] = w;
      }
    }
    __syncthreads();
    fft_row_smem<L, Q::E, INV, Q::GT>(sm + line * Q::LS, tid, tw, 1 + line);
    if constexpr (MID) {
      // row l = b2 holds X[b2 + C b1] at k = b1: times the symbol (stored
      // row-major [b2][b1] by th_symbol_layout), then back over b1 -> a1
      __syncthreads();
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int i = threadIdx.x + r * Q::THREADS;
        const int o = (i / L) * Q::LS + smem_pad(i % L);
        double2 w;
        if constexpr (SYM_SMEM) {
          w = sym_s[o];
        } else {
          w = io.th.sym[(l0 + i / L) * L + i % L];
          if (!io.th.transpose) w.y = -w.y;
        }
        sm[o] = cmul(sm[o], w);
      }
      __syncthreads();
      fft_row_smem<L, Q::E, !INV, Q::GT>(sm + line * Q::LS, tid, tw, 1 + line);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int i = threadIdx.x + r * Q::THREADS;
      const int j = rows_out ? i / L : i % LINES, k = rows_out ? i % L : i / LINES;
      const uint32_t l = l0 + j, lo = l & mmask, hi = l >> mshift;
      double2 x = sm[j * Q::LS + smem_pad(k)];
      if (mp.Q) {
        const uint32_t kk = (uint32_t)k;
        // exponent mod Q by masks (wrap-around of the 32-bit products is harmless mod 2^k)
        const uint32_t m = (lo * (hi * tu + kk * tv) + hi * kk * tz) & qmask;
        const double2 a = __ldg(&mp.twlo[m & ((1u << mp.twh) - 1u)]);
        const double2 b = __ldg(&mp.twhi[m >> mp.twh]);
        // w = a b = e^{-2 pi i m/Q}; the inverse direction uses its conjugate
        const double cs = a.x * b.x - a.y * b.y;
        double sn = a.x * b.y + a.y * b.x;
        if (TW_INV) sn = -sn;
        x = make_double2(x.x * cs - x.y * sn, x.x * sn + x.y * cs);
      }
      const uint32_t g = lo + hi * Hout + (uint32_t)k * Sout;
      dst_item[g] = x;
    }
  }
}

// The plain line pass with its first and last Stockham passes fused into the
// global load / store: a thread loads its first radix-8 butterfly's inputs
// x[tid + r L/8] straight from global memory, and (when the input and output
// layouts agree) stores its last pass's outputs straight to global memory --
// two of the per-element shared-memory round trips of fft_line_kernel saved
// (its passes were L1/shared-memory-bound: 87-96 % l1tex throughput).
// Threads are laid out line-minor for column passes (consecutive threads:
// consecutive lines, LINES x 16 B runs) and element-minor for row passes.
#ifndef FLB_LINE_MIN_CTAS_512
#define FLB_LINE_MIN_CTAS_512 2
#endif
template <int LOG2L, bool INV, bool PK = false>
__global__ void __launch_bounds__(LinePass<LOG2L>::THREADS,
                                  LinePass<LOG2L>::THREADS == 512 ? FLB_LINE_MIN_CTAS_512 : 0)
    fft_line_fused_kernel(const double2* __restrict__ src, double2* __restrict__ dst,
                          unsigned long long P, LineMap mp, const double2* __restrict__ tw,
                          NdctTrPack pk = NdctTrPack{}) {
  using Q = LinePass<LOG2L>;
  constexpr int L = Q::L, LINES = Q::LINES, TL = Q::TL, E = Q::E;
  constexpr int R0 = pass_radix(L, 1);
  static_assert(R0 == E, "one first-pass butterfly per thread");
  constexpr int NSL = last_pass_ns(L), RL = L / NSL;
  extern __shared__ double2 sm[];
  const uint32_t l0 = blockIdx.x * (uint32_t)LINES;
  const uint32_t mmask = (uint32_t)mp.M - 1u, qmask = (uint32_t)(mp.Q - 1);
  const int mshift = __ffsll((long long)mp.M) - 1;
  const uint32_t Hin = (uint32_t)mp.Hin, Sin = (uint32_t)mp.Sin, Hout = (uint32_t)mp.Hout,
                 Sout = (uint32_t)mp.Sout;
  const uint32_t tu = (uint32_t)mp.u, tv = (uint32_t)mp.v, tz = (uint32_t)mp.z;
  const bool rows_in = mp.Sin == 1, rows_out = mp.Sout == 1;
  const int t = threadIdx.x;
  const int line = rows_in ? t / TL : t % LINES;
  const int tid = rows_in ? t % TL : t / LINES;
  const size_t item = blockIdx.y;
  const double2* src_item = src + item * P;
  double2* dst_item = dst + item * P;
  double2* row = sm + line * Q::LS;
  const uint32_t lq = l0 + line, lo = lq & mmask, hi = lq >> mshift;
  auto out_twiddle = [&](uint32_t l_lo, uint32_t l_hi, uint32_t k, double2 x) {
    if (mp.Q) {
      const uint32_t m = (l_lo * (l_hi * tu + k * tv) + l_hi * k * tz) & qmask;
      const double2 a = __ldg(&mp.twlo[m & ((1u << mp.twh) - 1u)]);
      const double2 b = __ldg(&mp.twhi[m >> mp.twh]);
      const double cs = a.x * b.x - a.y * b.y;
      double sn = a.x * b.y + a.y * b.x;
      if (INV) sn = -sn;
      x = make_double2(x.x * cs - x.y * sn, x.x * sn + x.y * cs);
    }
    return x;
  };
  // first pass (NS = 1, no twiddles) from global memory
  double2 v[E];
  if constexpr (PK) {
    // the NDCT^T pack: entry m of row (tz, col) = wp[tz][m] (.) G[col][m]
    const size_t col = item % pk.nc, tz = item / pk.nc;
    const double2* G = pk.G + col * P;
    const double2* W = pk.wp + tz * P;
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const uint32_t g = lo + hi * Hin + (uint32_t)(tid + r * (L / R0)) * Sin;
      const double2 a = __ldg(&G[g]), w = __ldg(&W[g]);
      v[r] = make_double2(w.x * a.x, w.y * a.y);
    }
  } else {
#pragma unroll
    for (int r = 0; r < R0; ++r) v[r] = src_item[lo + hi * Hin + (uint32_t)(tid + r * (L / R0)) * Sin];
  }
  pass_compute<L, E, R0, 1, INV>(v, tid, tw);
  pass_store<L, E, R0, 1>(v, row, tid);
  __syncthreads();
  // middle passes in shared memory
  mid_passes<L, E, R0, NSL, INV, 0>(row, tid, tw, 0);
  // last pass
  pass_load<L, E, RL>(v, row, tid);
  pass_compute<L, E, RL, NSL, INV>(v, tid, tw + pass_tw_offset(L, NSL));
  if (rows_in == rows_out) {
#pragma unroll
    for (int q = 0; q < E / RL; ++q)
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const uint32_t k = (uint32_t)pass_out_index<L, E, RL, NSL>(tid, q, r);
        dst_item[lo + hi * Hout + k * Sout] = out_twiddle(lo, hi, k, v[q * RL + r]);
      }
  } else {
    // a transposing pass: through shared memory for a coalesced store
    __syncthreads();
    pass_store<L, E, RL, NSL>(v, row, tid);
    __syncthreads();
    constexpr int PER = LINES * L / Q::THREADS;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int i = t + r * Q::THREADS;
      const int j = rows_out ? i / L : i % LINES, k = rows_out ? i % L : i / LINES;
      const uint32_t l = l0 + j, llo = l & mmask, lhi = l >> mshift;
      dst_item[llo + lhi * Hout + (uint32_t)k * Sout] =
          out_twiddle(llo, lhi, (uint32_t)k, sm[j * Q::LS + smem_pad(k)]);
    }
  }
}

#ifndef FLB_FFT_FUSED
#define FLB_FFT_FUSED 1
#endif
template <int LOG2L, bool INV>
void launch_line_fused(const double2* src, double2* dst, unsigned long long P, size_t items,
                       const LineMap& mp, cudaStream_t s, const NdctTrPack* pk = nullptr) {
  using Q = LinePass<LOG2L>;
  const double2* tw = pass_twiddles(LOG2L);
  const unsigned long long lines = P >> LOG2L;
  LineMap m2 = mp;
  if (m2.Q) {
    const int lq = __builtin_ctzll(m2.Q);
    const auto t2 = twiddle_pair(lq);
    m2.twlo = t2.first;
    m2.twhi = t2.second;
    m2.twh = (lq + 1) / 2;
  }
  dim3 grid((unsigned)(lines / Q::LINES), (unsigned)items);
  if (pk) {
    auto kern = fft_line_fused_kernel<LOG2L, INV, true>;
    FLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM));
    kern<<<grid, Q::THREADS, Q::SMEM, s>>>(src, dst, P, m2, tw, *pk);
  } else {
    auto kern = fft_line_fused_kernel<LOG2L, INV>;
    FLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM));
    kern<<<grid, Q::THREADS, Q::SMEM, s>>>(src, dst, P, m2, tw, NdctTrPack{});
  }
  note_launch("fft_line_fused_kernel");
}

template <int LOG2L, bool INV, int IN, bool MID>
void launch_line(const LineIO& io, unsigned long long P, size_t items, const LineMap& mp,
                 cudaStream_t s) {
  using Q = LinePass<LOG2L>;
  static_assert(Q::LINES * Q::L == Q::THREADS * Q::E, "one element per thread per E");
  const double2* tw = pass_twiddles(LOG2L);
  const unsigned long long lines = P >> LOG2L;
  LineMap m2 = mp;
  if (m2.Q) {
    const int lq = __builtin_ctzll(m2.Q);
    const auto t2 = twiddle_pair(lq);
    m2.twlo = t2.first;
    m2.twhi = t2.second;
    m2.twh = (lq + 1) / 2;
  }
  auto kern = fft_line_kernel<LOG2L, INV, IN, MID>;
  // MID: + the symbol rows when they fit
  const size_t smem = MID && 2 * Q::SMEM <= 80 * 1024 ? 2 * Q::SMEM : Q::SMEM;
  FLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)(lines / Q::LINES), (unsigned)items);
  kern<<<grid, Q::THREADS, smem, s>>>(io, P, m2, tw);
  note_launch("fft_line_kernel");
}

template <bool INV, int IN = IO_PLAIN, bool MID = false>
void line_pass(int log2l, const LineIO& io, unsigned long long P, size_t items, const LineMap& mp,
               cudaStream_t s) {
  switch (log2l) {
    case 5: launch_line<5, INV, IN, MID>(io, P, items, mp, s); break;
    case 6: launch_line<6, INV, IN, MID>(io, P, items, mp, s); break;
    case 7: launch_line<7, INV, IN, MID>(io, P, items, mp, s); break;
    case 8: launch_line<8, INV, IN, MID>(io, P, items, mp, s); break;
    case 9: launch_line<9, INV, IN, MID>(io, P, items, mp, s); break;
    case 10: launch_line<10, INV, IN, MID>(io, P, items, mp, s); break;
    case 11: launch_line<11, INV, IN, MID>(io, P, items, mp, s); break;
    case 12: launch_line<12, INV, IN, MID>(io, P, items, mp, s); break;
    default: fail(FL_RUNTIME_ERROR, "fft: unsupported line length");
  }
}

template <bool INV>
void line_pass(int log2l, const double2* src, double2* dst, unsigned long long P, size_t items,
               const LineMap& mp, cudaStream_t s, const NdctTrPack* pk = nullptr) {
  if (FLB_FFT_FUSED || pk) {
    switch (log2l) {
      case 5: launch_line_fused<5, INV>(src, dst, P, items, mp, s, pk); return;
      case 6: launch_line_fused<6, INV>(src, dst, P, items, mp, s, pk); return;
      case 7: launch_line_fused<7, INV>(src, dst, P, items, mp, s, pk); return;
      case 8: launch_line_fused<8, INV>(src, dst, P, items, mp, s, pk); return;
      case 9: launch_line_fused<9, INV>(src, dst, P, items, mp, s, pk); return;
      case 10: launch_line_fused<10, INV>(src, dst, P, items, mp, s, pk); return;
      case 11: launch_line_fused<11, INV>(src, dst, P, items, mp, s, pk); return;
      case 12: launch_line_fused<12, INV>(src, dst, P, items, mp, s, pk); return;
      default: fail(FL_RUNTIME_ERROR, "fft: unsupported line length");
    }
  }
  LineIO io{};
  io.src = src;
  io.dst = dst;
  line_pass<INV>(log2l, io, P, items, mp, s);
}

// The pass plan: 2 passes for P <= 2^FLB_FFT_2PASS_MAX, else 3 (rows of
// 2^lr, columns of 2^lc = 2^l1 * 2^l2). Three passes of short lines (<= 2^8,
// eight lines per CTA: 128-byte column segments, several CTAs per SM) beat
// two of 2^11-2^12-point lines (one 1024-thread CTA per SM, 32-byte column
// segments) from P = 2^21: asymptotic conversion at N = 2^24 47.2 -> 40.3 ms,
// 2^22 10.6 -> 10.0 ms; equal at P = 2^19.
#ifndef FLB_FFT_2PASS_MAX
#define FLB_FFT_2PASS_MAX 20
#endif
#ifndef FLB_FFT_ROW_CEIL
#define FLB_FFT_ROW_CEIL 0  // 1: every odd log2p gives the longer line to the row pass
#endif
// (by default only 2^19: 512-point column lines, eight per CTA = 128-byte
// runs, and 1024-point contiguous rows instead of 1024-point columns in
// 64-byte runs: N = 2^20 DLT 1.74 -> 1.58 ms; at 2^15 and 2^17 the shorter
// row line wins: C2 0.495 vs 0.507 ms, 2^18 DLT 0.465 vs 0.484 ms)
struct PassPlan {
  int passes, lr, lc, l1, l2;
  unsigned long long R, C, C1, C2;
  explicit PassPlan(int log2p) {
    passes = (log2p <= FLB_FFT_2PASS_MAX || log2p < 15) ? 2 : 3;
    lr = passes == 2 ? (log2p + (FLB_FFT_ROW_CEIL || log2p == 19)) / 2 : log2p / 3;
    lc = log2p - lr;
    l1 = lc / 2;
    l2 = lc - l1;
    R = 1ull << lr;
    C = 1ull << lc;
    C1 = 1ull << l1;
    C2 = 1ull << l2;
  }
  // columns over a2 (stride R), twiddle w_P^{a1 b2}: -> a1 + R b2 (2 passes)
  LineMap col() const { return LineMap{R, 0, R, 0, R, twq(), 0, 1, 0}; }
  // over c2 (stride R C1), in place, twiddle w_C^{c1 d2}: lines l = a1 + R c1
  LineMap col1() const { return LineMap{R, R, R * C1, R, R * C1, C, 0, 0, 1}; }
  // over c1 (stride R) -> a1 + R (d2 + C2 d1), twiddle w_P^{a1 (d2 + C2 d1)};
  // lines l = a1 + R d2: lo = a1, hi = d2
  LineMap col2() const { return LineMap{R, R * C1, R, R, R * C2, twq(), 1, C2, 0}; }
  unsigned long long twq() const { return R * C; }
};

template <bool INV>
void fft_multipass(double2* d, double2* t, int log2p, size_t items, cudaStream_t s) {
  const unsigned long long P = 1ull << log2p;
  const PassPlan pp(log2p);
  if (pp.passes == 2) {
    line_pass<INV>(pp.lc, d, t, P, items, pp.col(), s);
  } else {
    line_pass<INV>(pp.l2, d, d, P, items, pp.col1(), s);
    line_pass<INV>(pp.l1, d, t, P, items, pp.col2(), s);
  }
  // rows over a1 (contiguous), written transposed to X[b2 + C b1]: lines l = b2
  line_pass<INV>(pp.lr, t, d, P, items, LineMap{1, pp.R, 1, 1, pp.C, 0, 0, 0, 0}, s);
}

// The last (row) pass of fft_multipass for the multi-pass NDCT, all terms of
// one column in one CTA with the unpack's weighted sum in registers
// (fft.cuh: NdctUnpack). Lines l = b2 (LINES adjacent ones per CTA) of the
// contiguous rows src[b2 R + a1]; output index m = b2 + C b1.
template <int LOG2L, bool INV>
__global__ void __launch_bounds__(LinePass<LOG2L>::THREADS)
    fft_row_unpack_kernel(const double2* __restrict__ src, unsigned long long P,
                          unsigned long long C, NdctUnpack a, const double2* __restrict__ tw) {
  using Q = LinePass<LOG2L>;
  constexpr int L = Q::L, LINES = Q::LINES, TL = Q::TL, E = Q::E;
  constexpr int R0 = pass_radix(L, 1);
  static_assert(R0 == E, "one first-pass butterfly per thread");
  constexpr int NSL = last_pass_ns(L), RL = L / NSL;
  constexpr int PER = LINES * L / Q::THREADS;
  extern __shared__ double2 sm[];
  const uint32_t l0 = blockIdx.x * (uint32_t)LINES;
  const int t = threadIdx.x;
  const int line = t / TL, tid = t % TL;
  const size_t col = blockIdx.y;
  double2* row = sm + line * Q::LS;
  double2 acc[PER];
#pragma unroll
  for (int r = 0; r < PER; ++r) acc[r] = make_double2(0.0, 0.0);
  const double2* src_line = src + col * P + (size_t)(l0 + line) * L + tid;
  const size_t term_stride = a.nc * P;
#pragma unroll 1
  for (int tz = 0; tz < a.nt; ++tz) {
    // the twiddle loads stay inside the loop (hoisted out of it they cost
    // ~150 registers: one CTA per SM)
    const double2* twi = tw;
    asm volatile("" : "+l"(twi));
    double2 v[E];
#pragma unroll
    for (int r = 0; r < R0; ++r) v[r] = src_line[(size_t)tz * term_stride + r * (L / R0)];
    pass_compute<L, E, R0, 1, INV>(v, tid, twi);
    pass_store<L, E, R0, 1>(v, row, tid);
    __syncthreads();
    mid_passes<L, E, R0, NSL, INV, 0>(row, tid, twi, 0);
    pass_load<L, E, RL>(v, row, tid);
    pass_compute<L, E, RL, NSL, INV>(v, tid, twi + pass_tw_offset(L, NSL));
    __syncthreads();
    pass_store<L, E, RL, NSL>(v, row, tid);
    __syncthreads();
    const double2* wp = a.wp + (size_t)tz * P;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int i = t + r * Q::THREADS;
      const int j = i % LINES, k = i / LINES;
      const double2 x = sm[j * Q::LS + smem_pad(k)];
      const double2 w = __ldg(&wp[(size_t)(l0 + j) + C * (size_t)k]);
      acc[r].x = __fma_rn(w.x, x.x, acc[r].x);
      acc[r].y = __fma_rn(w.y, x.y, acc[r].y);
    }
    __syncthreads();
  }
  double* o = a.out + col * a.ld;
  const size_t n2 = 4 * (size_t)P;  // 2N
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const int i = t + r * Q::THREADS;
    const int j = i % LINES, k = i / LINES;
    const size_t m = (size_t)(l0 + j) + C * (size_t)k;
    const size_t kx = m < P / 2 ? 4 * m : n2 - 4 * m - 1, ky = m < P / 2 ? 4 * m + 2 : n2 - 4 * m - 3;
    if (a.first) {
      o[kx] = acc[r].x;
      o[ky] = acc[r].y;
    } else {
      o[kx] += acc[r].x;
      o[ky] += acc[r].y;
    }
  }
}

template <int LOG2L, bool INV>
void launch_row_unpack(const double2* src, unsigned long long P, const NdctUnpack& a,
                       cudaStream_t s) {
  using Q = LinePass<LOG2L>;
  const double2* tw = pass_twiddles(LOG2L);
  const unsigned long long lines = P >> LOG2L;
  auto kern = fft_row_unpack_kernel<LOG2L, INV>;
  FLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM));
  dim3 grid((unsigned)(lines / Q::LINES), (unsigned)a.nc);
  kern<<<grid, Q::THREADS, Q::SMEM, s>>>(src, P, lines, a, tw);
  note_launch("fft_row_unpack_kernel");
}

template <bool INV>
void ndct_unpack_multipass(double2* d, double2* t, int log2p, const NdctUnpack& a, cudaStream_t s) {
  const unsigned long long P = 1ull << log2p;
  const PassPlan pp(log2p);
  const size_t items = (size_t)a.nt * a.nc;
  for (size_t b0 = 0; b0 < items; b0 += 65535) {
    const size_t nb = items - b0 < 65535 ? items - b0 : 65535;
    if (pp.passes == 2) {
      line_pass<INV>(pp.lc, d + b0 * P, t + b0 * P, P, nb, pp.col(), s);
    } else {
      line_pass<INV>(pp.l2, d + b0 * P, d + b0 * P, P, nb, pp.col1(), s);
      line_pass<INV>(pp.l1, d + b0 * P, t + b0 * P, P, nb, pp.col2(), s);
    }
  }
  switch (pp.lr) {
    case 7: launch_row_unpack<7, INV>(t, P, a, s); break;
    case 8: launch_row_unpack<8, INV>(t, P, a, s); break;
    case 9: launch_row_unpack<9, INV>(t, P, a, s); break;
    case 10: launch_row_unpack<10, INV>(t, P, a, s); break;
    default: fail(FL_RUNTIME_ERROR, "fft: unsupported row length for the fused unpack");
  }
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

template <bool INV>
void ndct_tr_pack_multipass(double2* d, double2* t, int log2p, const NdctTrPack& a, cudaStream_t s) {
  const unsigned long long P = 1ull << log2p;
  const PassPlan pp(log2p);
  const size_t items = (size_t)a.nt * a.nc;
  if (items > 65535) fail(FL_RUNTIME_ERROR, "fft: fused pack: too many rows");
  if (pp.passes == 2) {
    line_pass<INV>(pp.lc, d, t, P, items, pp.col(), s, &a);
  } else {
    line_pass<INV>(pp.l2, d, d, P, items, pp.col1(), s, &a);
    line_pass<INV>(pp.l1, d, t, P, items, pp.col2(), s);
  }
  line_pass<INV>(pp.lr, t, d, P, items, LineMap{1, pp.R, 1, 1, pp.C, 0, 0, 0, 0}, s);
}

void fft_pow2_ndct_tr_pack(double2* data, double2* scratch, int log2p, bool inverse,
                           const NdctTrPack& a, cudaStream_t s) {
  if (log2p <= kMaxSmemLog2 || log2p > kMaxLog2) fail(FL_RUNTIME_ERROR, "fft: fused pack: length");
  if (a.nc == 0 || a.nt == 0) return;
  if (inverse)
    ndct_tr_pack_multipass<true>(data, scratch, log2p, a, s);
  else
    ndct_tr_pack_multipass<false>(data, scratch, log2p, a, s);
}

bool fft_pow2_ndct_unpack_ok(int log2p) {
  if (log2p <= kMaxSmemLog2 || log2p > kMaxLog2) return false;
  const int lr = PassPlan(log2p).lr;
  return lr >= 7 && lr <= 10;
}

void fft_pow2_ndct_unpack(double2* data, double2* scratch, int log2p, bool inverse,
                          const NdctUnpack& a, cudaStream_t s) {
  if (!fft_pow2_ndct_unpack_ok(log2p)) fail(FL_RUNTIME_ERROR, "fft: fused unpack: length");
  if (a.nc == 0 || a.nt == 0) return;
  if (a.nc > 65535) fail(FL_RUNTIME_ERROR, "fft: fused unpack: too many columns");
  if (inverse)
    ndct_unpack_multipass<true>(data, scratch, log2p, a, s);
  else
    ndct_unpack_multipass<false>(data, scratch, log2p, a, s);
}

void th_symbol_layout(double2* sym, double2* scratch, int log2p, cudaStream_t s) {
  const PassPlan pp(log2p);
  // natural S[b2 + C b1] (R rows of C) -> [b2][b1]
  transpose(sym, scratch, (int)pp.R, (int)pp.C, 1, 0, false, s);
  FLB_CUDA(cudaMemcpyAsync(sym, scratch, (pp.R * pp.C) * sizeof(double2), cudaMemcpyDeviceToDevice,
                           s));
}

void th_sweep(const ThArgs& a, int log2p, size_t pairs, double2* V, double2* S, cudaStream_t s) {
  if (log2p <= kMaxSmemLog2 || log2p > kMaxLog2) fail(FL_RUNTIME_ERROR, "th_sweep: length");
  if (pairs == 0) return;
  if (pairs > 65535) fail(FL_RUNTIME_ERROR, "th_sweep: too many rank pairs");
  const unsigned long long P = 1ull << log2p;
  const PassPlan pp(log2p);
  LineIO io{};
  io.th = a;
  // forward columns, the first one packing V_q from x and the l_r rows
  if (pp.passes == 2) {
    io.dst = S;
    line_pass<false, IO_PACK>(pp.lc, io, P, pairs, pp.col(), s);
  } else {
    io.dst = V;
    line_pass<false, IO_PACK>(pp.l2, io, P, pairs, pp.col1(), s);
    io.src = V;
    io.dst = S;
    line_pass<false>(pp.l1, io, P, pairs, pp.col2(), s);
  }
  // rows b2 in place: forward over a1, times the symbol, inverse over b1,
  // twiddle w_P^{-a1 b2}
  io.src = S;
  io.dst = S;
  line_pass<false, IO_PLAIN, true>(pp.lr, io, P, pairs,
                                   LineMap{1, pp.R, 1, pp.R, 1, P, 0, 0, 1}, s);
  // inverse columns (natural b2 -> natural a2; the w_P twiddle is done)
  if (pp.passes == 3) line_pass<true>(pp.l2, io, P, pairs, pp.col1(), s);
  const int ll = pp.passes == 2 ? pp.lc : pp.l1;
  LineMap last = pp.passes == 2 ? pp.col() : pp.col2();
  last.Q = 0;
  io.dst = V;
  line_pass<true>(ll, io, P, pairs, last, s);
}

}  // namespace flb
