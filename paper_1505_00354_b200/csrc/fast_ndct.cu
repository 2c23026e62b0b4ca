// Fused Taylor NDCT on the cheb1 grid for power-of-two N: all L terms on
// chip, several columns per CTA.
//
// Replaces ndct.hpp:98-143 (L separate FFTW calls, each allocating and
// re-reading the column) on the hot path. Per column the kernel reads c once
// from HBM, keeps the stage vector (n/N)^l c_n in shared memory, runs the L
// real DCT-III (l even) / DST-III (l odd) transforms as N/2-point complex
// FFTs in shared memory (Makhoul's real-DCT packing), multiplies each by its
// Taylor weight sign_l (N delta_k)^l / l! in registers and writes f once:
// 16 B of HBM traffic per coefficient instead of the reference's ~48 B x L.
//
//   DST-III via DCT-III:  sum_n c_n sin(n t_k) = (-1)^k sum_{m>=1} c_{N-m} cos(m t_k)
//   DCT-III(a)_k, N even (t_k = (k+1/2) pi / N):
//     X_0 = a_0, X_j = a_j / 2, X_N = 0;  W_j = e^{i pi j/(2N)} (X_j - i X_{N-j})
//     Z_m = (W_m + W_{m+N/2}) + i (W_m - W_{m+N/2}) e^{2 pi i m/N},  m < N/2
//     z = IFFT_{N/2}(Z) (unnormalised);  w_{2m} = Re z_m, w_{2m+1} = Im z_m
//     y_{2n} = w_n,  y_{2n+1} = w_{N-1-n}
//   The transpose (ndct.hpp:121-143) is the mirror image: DCT-II through one
//   forward N/2-point FFT of the packed real sequence.
//
// Per term the packing feeds the first radix-8 FFT pass straight from
// registers, and (forward) the last pass is consumed in registers: each
// thread owns the 16 outputs its last-pass butterflies produce, so the Taylor
// weights are applied without another shared-memory round trip. The term
// parity (DCT/DST) is a template parameter.
//
// CTA layout: 256 threads = COLS groups of T = N/16 threads, one column per
// group, each group synchronising on its own named barrier so the columns of
// a CTA run out of phase. The column-independent tables -- N delta_k (in the
// order the weight updates read it) and the pass-major FFT twiddles -- are
// loaded into shared memory once per CTA. The stage vector is double-buffered:
// each term's pack reads its stage and writes the next term's, so the
// per-term stage update is one store per entry and no extra barrier phase.
//
// The same kernels with one unscaled term are the power-of-two cheb1
// dct_iii / dst_iii / *_transpose of trig.hpp (so ndct with zero
// perturbation stays bit-identical to dct_iii, test_ndct.cpp:112-125).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"
#include "fast_ndct.cuh"
#include "fft.cuh"
#include "launch.cuh"

namespace flb {

constexpr int kFastMinLog2 = 9;   // N = 512 (one warp per column)
constexpr int kFastMaxLog2 = 27;  // N <= 8192: one column per CTA; above: multi-pass (P <= 2^26)

struct FastNdct {
  size_t n = 0;
  int log2n = 0;
  int num_terms = 0;
  const double* delta = nullptr;  // cheb1 perturbations (device)
  double* owned_delta = nullptr;
  // Chebyshev (Jacobi-Anger) expansion of the same NDCT: bes_terms <
  // num_terms terms; weight / row tables [m][N] for the fused kernels
  // (N <= 8192), computed on the fly by the multi-pass kernels
  int bes_terms = 0;
  // swap: the sine flavour sum_n c_n sin(n theta_k) (dst_iii and its
  // transpose on a non-cheb1 grid): DCT and DST trade places per term and the
  // odd terms change sign (sin(a + b) = sin a cos b + cos a sin b)
  int swap = 0;
  cudaStream_t alloc_stream = nullptr;  // per-call objects: stream-ordered buffers
  bool async_alloc = false;
  double* bes_wf = nullptr;  // forward weights, owned-row order
  double* bes_wt = nullptr;  // transpose weights, tr_slot order
  double* bes_tt = nullptr;  // transpose row factors T_m(n/N), tr_row order
  double* cl_wf = nullptr;   // forward weights in the cluster kernel's thread order (2^14..2^16)
  // multi-pass path (N > 8192) of a plan-owned object: the weight / stage
  // tables [bes_terms][N] of all terms, kept after the first call (they
  // depend on the plan's offsets only; per call they cost 0.12 of 0.44 ms at
  // 2^20 and 14 of 25 ms at 2^26)
  mutable std::mutex big_mu;
  mutable double* big_wt = nullptr;
  mutable double* big_rt = nullptr;
  mutable double2* big_wp = nullptr;  // forward weights in packed-entry order (big_wp_kernel)
  mutable bool big_tried = false, big_wp_tried = false;
};

namespace {

__device__ __forceinline__ double taylor_sign_d(int l) { return ((l + 1) / 2) % 2 == 0 ? 1.0 : -1.0; }

template <int LOG2N>
struct Cfg {
  static constexpr int N = 1 << LOG2N;
  static constexpr int P = N / 2;
  static constexpr int E = 8;
  static constexpr int T = P / E;                 // threads per column
  static constexpr int OWN = N / T;               // rows owned per thread (= 2E)
// 256 threads per CTA measured faster than 512 at N = 4096 (24.3 vs 27.5 ms for
// 65536 columns, L = 17): the 255-register budget avoids the spills that the
// 128-register one forces (tools/bench_kernels.py, profiles/).
#ifndef FLB_NDCT_CTA_THREADS
#define FLB_NDCT_CTA_THREADS 256
#endif
  static constexpr int COLS = T >= FLB_NDCT_CTA_THREADS ? 1 : FLB_NDCT_CTA_THREADS / T;
  static constexpr int THREADS = T * COLS;
  static constexpr int TW = twiddle_entries(P);   // pass-major FFT twiddles
  static constexpr int NSL = last_pass_ns(P);     // last FFT pass
  static constexpr int RL = P / NSL;
  // per column: the stage vector double-buffered (term l reads one copy while
  // its pack writes term l+1's into the other) and the FFT row -- two of
  // them (ping-pong passes, one barrier per pass) when they fit beside the
  // tables (not at N = 8192)
  static constexpr size_t ZB = smem_row(P) * sizeof(double2);
  static constexpr bool PP = COLS * (2 * N * sizeof(double) + 2 * ZB) + N * 8 + TW * 16 <= 220 * 1024;
  static constexpr size_t COL_BYTES = 2 * N * sizeof(double) + (PP ? 2 : 1) * ZB;
  // tables in shared memory when they fit beside the columns
  static constexpr bool SMEM_TABLES = COLS * COL_BYTES + N * 8 + TW * 16 <= 220 * 1024;
  static constexpr int GT = COLS == 1 ? 0 : T;    // group barrier width (0 = whole CTA)
};

// The transpose kernel's layout. With the Chebyshev expansion (BES) it runs
// two CTAs per SM up to N = 4096 (<= 128 registers: the row factors are read
// where they are applied, no ping-pong rows, no shared tables): measured
// 28.3 -> 26.2 ms for the C4 IDLT. The Taylor transpose (row factors kept in
// registers) and the forward kernel are faster at one CTA per SM with
// ping-pong rows and shared tables.
#ifndef FLB_NDCT_TMEM
#define FLB_NDCT_TMEM 1
#endif
#ifndef FLB_NDCT_TR_PP
#define FLB_NDCT_TR_PP 1
#endif
#ifndef FLB_NDCT_TR_TMO
#define FLB_NDCT_TR_TMO 1
#endif
#ifndef FLB_NDCT_TR_T3
#define FLB_NDCT_TR_T3 1
#endif
constexpr int kTrCols = FLB_NDCT_TR_T3 ? 128 : 64;  // TMEM columns per CTA (NDCT^T, TMO)
#ifndef FLB_TM_FACC
#define FLB_TM_FACC 1  // TM forward kernel: the 16 accumulators per thread in TMEM too
#endif
#ifndef FLB_TM_WPF
#define FLB_TM_WPF 1  // TM forward kernel: the term's weights parked in TMEM (needs FACC's 256 columns)
#endif
constexpr int kTmCols = FLB_TM_FACC || FLB_TM_WPF ? 256 : 128;  // TMEM columns per CTA
template <int LOG2N, bool BES>
struct TrCfg {
  using C = Cfg<LOG2N>;
  static constexpr bool TWO = BES && LOG2N <= 12;
  // BES: the stage is the (weighted-on-the-fly) input itself, one buffer;
  // the Taylor stage's second buffer becomes a second FFT row (ping-pong)
  static constexpr bool ONE_STAGE = BES && TWO && FLB_NDCT_TR_PP && C::COLS == 1;
  static constexpr bool PP = ONE_STAGE || (!TWO && C::PP);
  // TMO: the output accumulators in TMEM (with ONE_STAGE)
  static constexpr bool TMO = ONE_STAGE && FLB_NDCT_TR_TMO;
  // T3: the input stage (read only by the pack) in TMEM too: shared memory
  // holds just the two FFT rows, three CTAs per SM
  static constexpr bool T3 = TMO && FLB_NDCT_TR_T3;
  static constexpr bool TABLES = !TWO && C::SMEM_TABLES;
  static constexpr int MINB = T3 ? 3 : TWO ? 2 : 1;
  static constexpr size_t COL_BYTES =
      (T3 ? 0 : ONE_STAGE ? 1 : 2) * C::N * sizeof(double) + (PP ? 2 : 1) * C::ZB;
  static constexpr size_t SMEM = C::COLS * COL_BYTES + (TABLES ? C::N * 8 + C::TW * 16 : 0);
};

#ifndef FLB_NDCT_FWD2
#define FLB_NDCT_FWD2 1
#endif
// The forward kernel's layout (TWO: two CTAs per SM as in TrCfg; with the
// Chebyshev expansion measured 26.0 -> 25.7 ms for the C4 DLT despite ~300 B
// of spills at the 128-register cap).
template <int LOG2N, bool BES>
struct FwdCfg {
  using C = Cfg<LOG2N>;
  static constexpr bool TWO = BES && FLB_NDCT_FWD2 && LOG2N <= 12;
  // TM (two CTAs per SM): the previous Chebyshev stage T_{m-1}(x) c -- read
  // only at a thread's own entries -- lives in tensor memory, which frees
  // the second shared stage buffer for a second FFT row (ping-pong passes)
  static constexpr bool TM = TWO && FLB_NDCT_TMEM && C::COLS == 1;
  static constexpr int MINB = TWO ? 2 : 1;
  static constexpr bool PP = TM || (!TWO && C::PP);
  static constexpr bool TABLES = !TWO && C::SMEM_TABLES;
  static constexpr size_t COL_BYTES = (TM ? 1 : 2) * C::N * sizeof(double) + (PP ? 2 : 1) * C::ZB;
  static constexpr size_t SMEM = C::COLS * COL_BYTES + (TABLES ? C::N * 8 + C::TW * 16 : 0);
};

// Output row k of w index q (q = 2m or 2m+1 of the inverse FFT output z_m).
template <int N>
__device__ __forceinline__ int fwd_row_of(int q) {
  return q < N / 2 ? 2 * q : 2 * (N - 1 - q) + 1;
}

// Shared-memory slot of output row k when a column's outputs are staged for
// a coalesced store: the rows a half-warp scatters are 4 apart (k = 4m + c,
// consecutive m), four per 16 banks of doubles; XOR-ing bits 0-1 with bits
// 4-5 spreads them over all 16 (the staging stores were 4-way conflicted,
// 20% of the plain DCT pass's shared-memory wavefronts), and the row-order
// reads (16 consecutive k) stay conflict-free. A permutation within each
// aligned group of 4.
__device__ __forceinline__ int out_slot(int k) { return k ^ ((k >> 4) & 3); }

// e^{i pi r/32} and e^{i pi r/8}, r < 8: with T = N/16 threads per column the
// pack twiddles of m = t + r T are per-thread bases times these constants.
// (16 entries: the transpose's unpack uses rows n = t + i T, i < 16.)
struct PackConst {
  static constexpr double c32[16][2] = {
      {1.0, 0.0}, {0.9951847266721969, 0.0980171403295606}, {0.9807852804032304, 0.19509032201612828},
      {0.9569403357322088, 0.2902846772544624}, {0.9238795325112867, 0.3826834323650898},
      {0.881921264348355, 0.47139673682599764}, {0.8314696123025452, 0.5555702330196022},
      {0.773010453362737, 0.6343932841636455}, {0.7071067811865476, 0.7071067811865476},
      {0.6343932841636455, 0.773010453362737}, {0.5555702330196022, 0.8314696123025452},
      {0.47139673682599764, 0.881921264348355}, {0.3826834323650898, 0.9238795325112867},
      {0.2902846772544624, 0.9569403357322088}, {0.19509032201612828, 0.9807852804032304},
      {0.0980171403295606, 0.9951847266721969}};
  static constexpr double c8[16][2] = {
      {1.0, 0.0}, {0.9238795325112867, 0.3826834323650898}, {0.7071067811865476, 0.7071067811865476},
      {0.3826834323650898, 0.9238795325112867}, {0.0, 1.0}, {-0.3826834323650898, 0.9238795325112867},
      {-0.7071067811865476, 0.7071067811865476}, {-0.9238795325112867, 0.3826834323650898},
      {-1.0, 0.0}, {-0.9238795325112867, -0.3826834323650898}, {-0.7071067811865476, -0.7071067811865476},
      {-0.3826834323650898, -0.9238795325112867}, {0.0, -1.0}, {0.3826834323650898, -0.9238795325112867},
      {0.7071067811865476, -0.7071067811865476}, {0.9238795325112867, -0.3826834323650898}};
};

// The same constants in constant memory, for loop-indexed use.
__constant__ double kC32[16][2] = {
    {1.0, 0.0}, {0.9951847266721969, 0.0980171403295606}, {0.9807852804032304, 0.19509032201612828},
    {0.9569403357322088, 0.2902846772544624}, {0.9238795325112867, 0.3826834323650898},
    {0.881921264348355, 0.47139673682599764}, {0.8314696123025452, 0.5555702330196022},
    {0.773010453362737, 0.6343932841636455}, {0.7071067811865476, 0.7071067811865476},
    {0.6343932841636455, 0.773010453362737}, {0.5555702330196022, 0.8314696123025452},
    {0.47139673682599764, 0.881921264348355}, {0.3826834323650898, 0.9238795325112867},
    {0.2902846772544624, 0.9569403357322088}, {0.19509032201612828, 0.9807852804032304},
    {0.0980171403295606, 0.9951847266721969}};
__constant__ double kC8[16][2] = {
    {1.0, 0.0}, {0.9238795325112867, 0.3826834323650898}, {0.7071067811865476, 0.7071067811865476},
    {0.3826834323650898, 0.9238795325112867}, {0.0, 1.0}, {-0.3826834323650898, 0.9238795325112867},
    {-0.7071067811865476, 0.7071067811865476}, {-0.9238795325112867, 0.3826834323650898},
    {-1.0, 0.0}, {-0.9238795325112867, -0.3826834323650898}, {-0.7071067811865476, -0.7071067811865476},
    {-0.3826834323650898, -0.9238795325112867}, {0.0, -1.0}, {0.3826834323650898, -0.9238795325112867},
    {0.7071067811865476, -0.7071067811865476}, {0.9238795325112867, -0.3826834323650898}};

// The pack arithmetic from the four stage values (stage[m], stage[m + P],
// stage[N - m], stage[P - m]); m0: m == 0.
template <bool ODD, int R, bool HALF = false>
__device__ __forceinline__ double2 fwd_pack_vals(double s_m, double s_mp, double s_nm, double s_pm,
                                                 bool m0, double2 ta_t, double2 r4_t) {
  constexpr double h = 0.70710678118654752440;
  // X_j = a_j / 2 (X_0 = a_0, X_N = 0); a = stage (DCT) or the reversed stage (DST)
  constexpr double hf = HALF ? 1.0 : 0.5;  // (multiplications by 1.0 fold away)
  const double xa = ODD ? (m0 ? 0.0 : hf * s_nm) : (m0 ? (HALF ? 2.0 * s_m : s_m) : hf * s_m);
  const double xan = m0 ? 0.0 : hf * (ODD ? s_m : s_nm);
  const double xb = hf * (ODD ? s_pm : s_mp);
  const double xbn = hf * (ODD ? s_mp : s_pm);
  constexpr double a32x = PackConst::c32[R][0], a32y = PackConst::c32[R][1];
  constexpr double a8x = PackConst::c8[R][0], a8y = PackConst::c8[R][1];
  // e^{i pi m/(2N)}, e^{i pi (m+P)/(2N)} = e^{i pi/4} e^{i pi m/(2N)}, e^{2 pi i m/N}
  const double2 ta = make_double2(ta_t.x * a32x - ta_t.y * a32y, ta_t.x * a32y + ta_t.y * a32x);
  const double2 tb = make_double2(h * (ta.x - ta.y), h * (ta.x + ta.y));
  const double2 r4 = make_double2(r4_t.x * a8x - r4_t.y * a8y, r4_t.x * a8y + r4_t.y * a8x);
  const double2 Wa = make_double2(ta.x * xa + ta.y * xan, ta.y * xa - ta.x * xan);
  const double2 Wb = make_double2(tb.x * xb + tb.y * xbn, tb.y * xb - tb.x * xbn);
  const double2 s = make_double2(Wa.x + Wb.x, Wa.y + Wb.y);
  const double2 d = make_double2(Wa.x - Wb.x, Wa.y - Wb.y);
  const double2 dr = make_double2(d.x * r4.x - d.y * r4.y, d.x * r4.y + d.y * r4.x);
  return make_double2(s.x - dr.y, s.y + dr.x);  // s + i dr
}

// Packed Z_m of the forward transform for term parity ODD, m = t + r T.
// ta_t = e^{i pi t/(2N)}, r4_t = e^{2 pi i t/N} (per-thread bases).
// The pack of Z_m reads stage entries {m, m + P, N - m, P - m} (both term
// parities); with NEXT the thread also writes its own two, m and m + P, scaled
// by n/N into `next` -- the stage of the following term -- so the stage
// update costs one store per entry and no separate pass.
// NM: 0 = no next stage; 1 = next = x c (Taylor (n/N)^{l+1} c_n, and the
// Chebyshev T_1); 2 = next = 2 x cur - next (Chebyshev T_{m+1}(x) c_n, the
// buffer `next` holding T_{m-1}(x) c_n), x = n/N.
// bad (optional): set when stage[m] or stage[m + P] is not finite (every entry
// is some thread's m or m + P), so a caller needs no separate check pass.
// HALF: the stage holds a/2 (the 1/2 of X_j = a_j/2 pre-applied), saving
// four multiplies per Z.
template <int N, bool ODD, int R, int NM, bool HALF = false>
__device__ __forceinline__ double2 fwd_pack(const double* stage, double* next, int m, double2 ta_t,
                                            double2 r4_t, bool* bad = nullptr,
                                            double2* own = nullptr) {
  constexpr int P = N / 2;
  const double s_m = stage[m], s_mp = stage[m + P];
  if (own) *own = make_double2(s_m, s_mp);
  if (bad) *bad |= !isfinite(s_m) || !isfinite(s_mp);
  const double s_nm = stage[(N - m) & (N - 1)], s_pm = stage[P - m];
  if (NM == 1) {
    next[m] = s_m * ((double)m / (double)N);  // (n/N)^{l+1} c_n
    next[m + P] = s_mp * ((double)(m + P) / (double)N);
  } else if (NM == 2) {
    next[m] = fma(2.0 * ((double)m / (double)N), s_m, -next[m]);
    next[m + P] = fma(2.0 * ((double)(m + P) / (double)N), s_mp, -next[m + P]);
  }
  return fwd_pack_vals<ODD, R, HALF>(s_m, s_mp, s_nm, s_pm, m == 0, ta_t, r4_t);
}

// The rows thread t of the forward kernel accumulates: the outputs of its
// last-pass butterflies (i < OWN).
template <int LOG2N>
__device__ __forceinline__ int fwd_own_row(int t, int i) {
  using C = Cfg<LOG2N>;
  const int s = i >> 1, q = s / C::RL, r = s % C::RL;
  return fwd_row_of<C::N>(2 * (t + q * C::T + r * C::NSL) + (i & 1));
}

// One forward Taylor term (or one plain transform): f[i] += sign p[i] y_{k_i}.
template <int N, bool ODD, int NM, int R, bool SPLIT = false>
__device__ __forceinline__ void fwd_pack_all(double2* v, const double* stage, double* next, int t,
                                             double2 ta_t, double2 r4_t, bool* bad = nullptr) {
  if constexpr (SPLIT && R == 4) asm volatile("" ::: "memory");  // two halves: fewer live loads
  if constexpr (R < 8) {
    v[R] = fwd_pack<N, ODD, R, NM>(stage, next, t + R * (N / 16), ta_t, r4_t, bad);
    fwd_pack_all<N, ODD, NM, R + 1, SPLIT>(v, stage, next, t, ta_t, r4_t, bad);
  }
}

// One forward Taylor term (or one plain transform): f[i] += sign p[i] y_{k_i}.
// The first pass stores into zx. Ping-pong (C::PP): the passes alternate
// between zx and zy; the caller passes, as the next term's zx, the buffer the
// last pass did NOT read (returned: the one it read), so no barrier is needed
// before the first store. In place: a barrier orders the first store after
// the previous term's last-pass reads.
template <int LOG2N, bool ODD, int NM, bool PPX = Cfg<LOG2N>::PP, int PST = 1, bool SPLIT = false>
__device__ __forceinline__ double2* fwd_term(const double* stage, double* next, double2* zx,
                                             double2* zy, int t, int bar, double2 ta_t,
                                             double2 r4_t, const double2* fftw, const double* p,
                                             double* f, double sign) {
  using C = Cfg<LOG2N>;
  constexpr int N = C::N, P = C::P, T = C::T, E = C::E, NSL = C::NSL, RL = C::RL;
  static_assert(E == 8 && T == N / 16, "pack twiddle constants assume T = N/16");
  double2 v[E];
  fwd_pack_all<N, ODD, NM, 0, SPLIT>(v, stage, next, t, ta_t, r4_t);
  pass_compute<P, E, 8, 1, true>(v, t, fftw);
  double2* fin = zx;
  if constexpr (PPX) {
    pass_store<P, E, 8, 1>(v, zx, t);
    group_sync<C::GT>(bar);
    fin = mid_passes_pp<P, E, 8, NSL, true, C::GT, true>(zx, zy, t, fftw, bar);
  } else {
    group_sync<C::GT>(bar);
    pass_store<P, E, 8, 1>(v, zx, t);
    group_sync<C::GT>(bar);
    mid_passes<P, E, 8, NSL, true, C::GT, true>(zx, t, fftw, bar);
  }
  pass_load<P, E, RL>(v, fin, t);
  pass_compute<P, E, RL, NSL, true, true>(v, t, fftw + pass_tw_offset(P, NSL));
#pragma unroll
  for (int q = 0; q < E / RL; ++q)
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const int m = t + q * T + r * NSL;
      const double2 z = v[q * RL + r];
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const int i = 2 * (q * RL + r) + part;
        const int k = fwd_row_of<N>(2 * m + part);
        double y = part ? z.y : z.x;
        if (ODD && (k & 1)) y = -y;
        const double w = PST == 1 ? p[i] : __ldg(p + i * PST);  // PST > 1: a global row
        f[i] += sign * w * y;
      }
    }
  return fin;
}

// ---- tensor-memory stage (FwdCfg::TM) --------------------------------------
// Each thread keeps 16 doubles of its own stage entries (m, m + P for its 8
// m) per slot in its TMEM lane: slot A = T_{m-1}(x) c, slot B = the next
// stage T_{m+1}(x) c until it is written back to shared memory.
__device__ __forceinline__ void tm_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_ld8_nw(uint32_t taddr, uint32_t* v) {  // caller waits
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void split2(double d, uint32_t* w) {
  w[0] = (uint32_t)__double2loint(d);
  w[1] = (uint32_t)__double2hiint(d);
}
__device__ __forceinline__ double join2(const uint32_t* w) {
  return __hiloint2double((int)w[1], (int)w[0]);
}

// Half h (entries r = 4h .. 4h + 3) of the TM pack: Z_m for m = t + r T from
// the shared stage T_l c (own and mirrored entries), and at the own entries
// next = x c (FIRST) or 2 x T_l c - T_{l-1} c; T_l c -> slot A, next -> B.
// The stage holds T_l(x) c / 2 (fwd_pack HALF; the recurrence is linear).
// xt2 = 2 t / N: 2 x_m = xt2 + R/8 and 2 x_{m+P} = 2 x_m + 1 (m = t + R N/16).
template <int N, bool ODD, bool FIRST, int R, int RE>
__device__ __forceinline__ void tm_pack_rec(double2* v, const double* stage, int t, double xt2,
                                            double2 ta_t, double2 r4_t,
                                            const uint32_t (&prev)[8], uint32_t (&cw)[8],
                                            uint32_t (&nw)[8]) {
  if constexpr (R < RE) {
    constexpr int rr = R % 2;
    const int m = t + R * (N / 16);
    double2 own;
    v[R] = fwd_pack<N, ODD, R, 0, true>(stage, nullptr, m, ta_t, r4_t, nullptr, &own);
    const double tx0 = xt2 + (double)R / 8.0, tx1 = tx0 + 1.0;  // 2 x (exact)
    double n0, n1;
    if constexpr (FIRST) {
      n0 = own.x * (0.5 * tx0);
      n1 = own.y * (0.5 * tx1);
    } else {
      n0 = fma(tx0, own.x, -join2(&prev[4 * rr]));
      n1 = fma(tx1, own.y, -join2(&prev[4 * rr + 2]));
    }
    split2(own.x, &cw[4 * rr]);
    split2(own.y, &cw[4 * rr + 2]);
    split2(n0, &nw[4 * rr]);
    split2(n1, &nw[4 * rr + 2]);
    tm_pack_rec<N, ODD, FIRST, R + 1, RE>(v, stage, t, xt2, ta_t, r4_t, prev, cw, nw);
  }
}

// One Chebyshev term of the TM forward kernel (PST = T weights, ping-pong
// FFT rows zx / zy): returns the row the last pass read.
template <int LOG2N, bool ODD, bool FIRST>
__device__ __forceinline__ double2* tm_fwd_term(double* stage, double2* zx, double2* zy, int t,
                                                double2 ta_t, double2 r4_t, const double2* fftw,
                                                const double* p, double* f, uint32_t tA,
                                                uint32_t tB, uint32_t tF, uint32_t tW) {
  using C = Cfg<LOG2N>;
  constexpr int N = C::N, P = C::P, T = C::T, E = C::E, NSL = C::NSL, RL = C::RL;
  static_assert(E == 8 && T == N / 16, "pack twiddle constants assume T = N/16");
  constexpr int PST = T;
  const double xt2 = (double)(2 * t) / (double)N;
  double2 v[E];
  // quarters (two entries r each): few live registers around the pack
#define FLB_TM_QUARTER(Q)                                                                   \
  {                                                                                         \
    uint32_t prev[8], cw[8], nw[8];                                                         \
    if constexpr (!FIRST) tm_ld8(tA + 8 * (Q), prev);                                       \
    tm_pack_rec<N, ODD, FIRST, 2 * (Q), 2 * (Q) + 2>(v, stage, t, xt2, ta_t, r4_t, prev, cw, nw); \
    tm_st8(tA + 8 * (Q), cw);                                                               \
    tm_st8(tB + 8 * (Q), nw);                                                               \
  }
  // FLB_TM_WPF: the term's 16 weights are loaded now (L2) and parked in TMEM
  // slot W after the pack, so the unpack reads them without a global round trip
  double wq[FLB_TM_WPF ? 16 : 1];
  if constexpr (FLB_TM_WPF) {
#pragma unroll
    for (int i = 0; i < 16; ++i) wq[i] = __ldg(p + i * PST);
  }
  FLB_TM_QUARTER(0)
  FLB_TM_QUARTER(1)
  FLB_TM_QUARTER(2)
  FLB_TM_QUARTER(3)
#undef FLB_TM_QUARTER
  if constexpr (FLB_TM_WPF) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      uint32_t ww[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) split2(wq[4 * h + j], &ww[2 * j]);
      tm_st8(tW + 8 * h, ww);
    }
  }
  pass_compute<P, E, 8, 1, true>(v, t, fftw);
  pass_store<P, E, 8, 1>(v, zx, t);
  tm_wait_st();
  __syncthreads();  // pass-1 rows complete; every pack has read the stage
  // write the next stage back over this one (own entries)
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    uint32_t nw[8];
    tm_ld8(tB + 8 * h, nw);
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int m = t + (2 * h + rr) * T;
      stage[m] = join2(&nw[4 * rr]);
      stage[m + P] = join2(&nw[4 * rr + 2]);
    }
  }
  double2* fin = mid_passes_pp<P, E, 8, NSL, true, 0, true>(zx, zy, t, fftw, 0);
  pass_load<P, E, RL>(v, fin, t);
  pass_compute<P, E, RL, NSL, true, true>(v, t, fftw + pass_tw_offset(P, NSL));
  if constexpr (FLB_TM_FACC) {
    // the accumulators live in TMEM (slot F): load, update, store back
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t fw[16], wv[16];
      tm_ld8(tF + 16 * h, fw);
      tm_ld8(tF + 16 * h + 8, fw + 8);
      if constexpr (FLB_TM_WPF) {
        tm_ld8(tW + 16 * h, wv);
        tm_ld8(tW + 16 * h + 8, wv + 8);
      }
#pragma unroll
      for (int i8 = 0; i8 < 8; ++i8) {
        const int i = 8 * h + i8, s = i >> 1, q = s / RL, r = s % RL, part = i & 1;
        const int m = t + q * T + r * NSL;
        const double2 z = v[q * RL + r];
        const int k = fwd_row_of<N>(2 * m + part);
        double y = part ? z.y : z.x;
        if (ODD && (k & 1)) y = -y;
        const double w = FLB_TM_WPF ? join2(&wv[2 * i8]) : __ldg(p + i * PST);
        split2(join2(&fw[2 * i8]) + w * y, &fw[2 * i8]);
      }
      tm_st8(tF + 16 * h, fw);
      tm_st8(tF + 16 * h + 8, fw + 8);
    }
  } else {
#pragma unroll
    for (int q = 0; q < E / RL; ++q)
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int m = t + q * T + r * NSL;
        const double2 z = v[q * RL + r];
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          const int i = 2 * (q * RL + r) + part;
          const int k = fwd_row_of<N>(2 * m + part);
          double y = part ? z.y : z.x;
          if (ODD && (k & 1)) y = -y;
          f[i] += __ldg(p + i * PST) * y;
        }
      }
  }
  return fin;
}

// plain_op: -1 = NDCT with num_terms terms; 0 = one plain DCT-III;
// 1 = one plain DST-III. BES: Chebyshev (Jacobi-Anger) expansion instead of
// Taylor -- stage T_m(n/N) c_n by the three-term recurrence, weights
// wtab[m][i T + t] (sign included) of the thread's owned rows from a table.
template <int LOG2N, bool BES>
__global__ void __launch_bounds__(Cfg<LOG2N>::THREADS, FwdCfg<LOG2N, BES>::MINB)
    fast_ndct_fwd_kernel(const double* __restrict__ in, size_t ld_in, double* __restrict__ out,
                         size_t ld_out, size_t batch, const double* __restrict__ delta,
                         int num_terms, int plain_op, const double2* __restrict__ tw4n,
                         const double2* __restrict__ fftw_g, const double* __restrict__ wtab,
                         int* nonfinite, int swap) {
  using C = Cfg<LOG2N>;
  using FC = FwdCfg<LOG2N, BES>;
  constexpr int N = C::N, T = C::T, OWN = C::OWN;
  extern __shared__ double smem[];
  double* nd = smem + C::COLS * (FC::COL_BYTES / 8);
  double2* fftw_s = reinterpret_cast<double2*>(nd + N);
  const double2* fftw = FC::TABLES ? fftw_s : fftw_g;
  auto own_row = [](int t, int i) -> int { return fwd_own_row<LOG2N>(t, i); };
  if (FC::TABLES) {
    // N delta in owned-row order, nd[i T + t] for row own_row(t, i): the
    // per-term weight update reads it conflict-free (row order is stride 4)
    if (plain_op < 0 && !BES)
      for (int j = threadIdx.x; j < N; j += blockDim.x)
        nd[j] = (double)N * delta[own_row(j % T, j / T)];
    load_table(fftw_s, fftw_g, C::TW);
    __syncthreads();
  }
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int bar = 1 + g;
  const size_t col = (size_t)blockIdx.x * C::COLS + g;
  if (col >= batch) return;
  double* stage = smem + g * (FC::COL_BYTES / 8);  // (n/N)^l c_n, terms l even
  double* stage_odd = stage + N;                  // terms l odd (not with TM)
  double2* zbA = reinterpret_cast<double2*>(stage + (FC::TM ? 1 : 2) * N);
  double2* zbB = FC::PP ? zbA + C::ZB / sizeof(double2) : zbA;
  double2* zx = zbA;  // the first pass's target this term
  auto other = [&](double2* b) { return b == zbA ? zbB : zbA; };
  const double* src = in + col * ld_in;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < OWN; ++i) {
    const int n = t + T * i;
    const double v = src[n];
    bad |= !isfinite(v);
    // the TM Chebyshev path keeps the stage halved (fwd_pack HALF)
    stage[n] = (BES && FC::TM && plain_op < 0) ? 0.5 * v : v;
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
  auto kown = [&](int i) -> int { return own_row(t, i); };
  double f[OWN], p[OWN];
#pragma unroll
  for (int i = 0; i < OWN; ++i) {
    f[i] = 0.0;
    p[i] = 1.0;
  }
  // per-thread pack twiddle bases e^{i pi t/(2N)}, e^{2 pi i t/N} (table of 4N-th roots)
  const double2 ta_t = __ldg(&tw4n[t]);
  const double2 r4_t = __ldg(&tw4n[4 * t]);
  group_sync<C::GT>(bar);
  if (plain_op >= 0) {
    if (plain_op == 1)
      fwd_term<LOG2N, true, 0, FC::PP>(stage, nullptr, zx, other(zx), t, bar, ta_t, r4_t, fftw, p, f, 1.0);
    else
      fwd_term<LOG2N, false, 0, FC::PP>(stage, nullptr, zx, other(zx), t, bar, ta_t, r4_t, fftw, p, f, 1.0);
  } else if (BES && FC::TM) {
    // previous stage in TMEM, ping-pong FFT rows (FwdCfg::TM)
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base))),
                   "n"(kTmCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // this warp's lane quarter; per warp 64 (+ 32 with FLB_TM_FACC) columns
    constexpr uint32_t kWarpCols = FLB_TM_FACC || FLB_TM_WPF ? 128u : 64u;
    const uint32_t tA = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + kWarpCols * (uint32_t)(warp >> 2);
    const uint32_t tB = tA + 32;
    const uint32_t tF = tA + 64;
    const uint32_t tW = tA + 96;  // (FLB_TM_WPF)
    if constexpr (FLB_TM_FACC) {
      uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int q = 0; q < 4; ++q) tm_st8(tF + 8 * q, z);
      tm_wait_st();
    }
    double2* zy = zbB;
    for (int m = 0; m < num_terms; ++m) {
      const double* wr = wtab + (size_t)m * N + t;
      double2* fin;
      if (m == 0 && swap)
        fin = tm_fwd_term<LOG2N, true, true>(stage, zx, zy, t, ta_t, r4_t, fftw, wr, f, tA, tB, tF, tW);
      else if (m == 0)
        fin = tm_fwd_term<LOG2N, false, true>(stage, zx, zy, t, ta_t, r4_t, fftw, wr, f, tA, tB, tF, tW);
      else if ((m & 1) ^ swap)
        fin = tm_fwd_term<LOG2N, true, false>(stage, zx, zy, t, ta_t, r4_t, fftw, wr, f, tA, tB, tF, tW);
      else
        fin = tm_fwd_term<LOG2N, false, false>(stage, zx, zy, t, ta_t, r4_t, fftw, wr, f, tA, tB, tF, tW);
      zy = fin;  // the next term's first pass writes the row the last pass did not read
      zx = other(fin);
    }
    if constexpr (FLB_TM_FACC) {
      tm_wait_st();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t fw[8];
        tm_ld8(tF + 8 * q, fw);
#pragma unroll
        for (int j = 0; j < 4; ++j) f[4 * q + j] = join2(&fw[2 * j]);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(kTmCols)
                   : "memory");
  } else if (BES && FC::TWO) {
    // weights read where they are applied (PST = T), pack in two halves
    for (int m = 0; m < num_terms; ++m) {
      const double* wr = wtab + (size_t)m * N + t;
      if (m == 0 && swap)
        fwd_term<LOG2N, true, 1, false, T, true>(stage, stage_odd, zx, zx, t, bar, ta_t, r4_t,
                                                 fftw, wr, f, 1.0);
      else if (m == 0)
        fwd_term<LOG2N, false, 1, false, T, true>(stage, stage_odd, zx, zx, t, bar, ta_t, r4_t,
                                                  fftw, wr, f, 1.0);
      else if (swap && (m & 1))  // sine flavour: a DCT of the odd-m stage
        fwd_term<LOG2N, false, 2, false, T, true>(stage_odd, stage, zx, zx, t, bar, ta_t, r4_t,
                                                  fftw, wr, f, 1.0);
      else if (swap)  // m even, sine flavour: a DST of the even-m stage
        fwd_term<LOG2N, true, 2, false, T, true>(stage, stage_odd, zx, zx, t, bar, ta_t, r4_t,
                                                 fftw, wr, f, 1.0);
      else if (m & 1)
        fwd_term<LOG2N, true, 2, false, T, true>(stage_odd, stage, zx, zx, t, bar, ta_t, r4_t,
                                                 fftw, wr, f, 1.0);
      else
        fwd_term<LOG2N, false, 2, false, T, true>(stage, stage_odd, zx, zx, t, bar, ta_t, r4_t,
                                                  fftw, wr, f, 1.0);
    }
  } else if (BES) {
    for (int m = 0; m < num_terms; ++m) {
#pragma unroll
      for (int i = 0; i < OWN; ++i) p[i] = __ldg(wtab + (size_t)m * N + i * T + t);
      double2* fin;
      if (m == 0 && swap)
        fin = fwd_term<LOG2N, true, 1, FC::PP>(stage, stage_odd, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                                       p, f, 1.0);
      else if (m == 0)
        fin = fwd_term<LOG2N, false, 1, FC::PP>(stage, stage_odd, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                                        p, f, 1.0);
      else if (swap && (m & 1))  // sine flavour: a DCT of the odd-m stage
        fin = fwd_term<LOG2N, false, 2, FC::PP>(stage_odd, stage, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                                        p, f, 1.0);
      else if (swap)
        fin = fwd_term<LOG2N, true, 2, FC::PP>(stage, stage_odd, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                                       p, f, 1.0);
      else if (m & 1)
        fin = fwd_term<LOG2N, true, 2, FC::PP>(stage_odd, stage, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                                       p, f, 1.0);
      else
        fin = fwd_term<LOG2N, false, 2, FC::PP>(stage, stage_odd, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                                        p, f, 1.0);
      zx = other(fin);
    }
  } else {
    for (int l = 0; l < num_terms; ++l) {
      if (l > 0) {
        const double inv_l = 1.0 / (double)l;
#pragma unroll
        for (int i = 0; i < OWN; ++i) {
          const double q = FC::TABLES ? nd[i * T + t] : (double)N * __ldg(&delta[kown(i)]);
          p[i] *= q * inv_l;  // (N delta_k)^l / l!
        }
      }
      double2* fin;
      if (l & 1)
        fin = fwd_term<LOG2N, true, 1, FC::PP>(stage_odd, stage, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                                       p, f, taylor_sign_d(l));
      else
        fin = fwd_term<LOG2N, false, 1, FC::PP>(stage, stage_odd, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                                        p, f, taylor_sign_d(l));
      zx = other(fin);
    }
  }
  // scatter the owned rows through shared memory, then one coalesced store
  group_sync<C::GT>(bar);
#pragma unroll
  for (int i = 0; i < OWN; ++i) stage[out_slot(kown(i))] = f[i];
  group_sync<C::GT>(bar);
  double* dst = out + col * ld_out;
#pragma unroll
  for (int i = 0; i < OWN; ++i) dst[t + T * i] = stage[out_slot(t + T * i)];
}

// Layout of the transposed stage h in shared memory: even entries first,
// hs[q] = h_{2q}, hs[P + q] = h_{2q+1}, so the pack below reads contiguous
// pairs (row order would be a stride-4, 4-way bank-conflicted read).
template <int N>
__device__ __forceinline__ int tr_slot(int k) { return (k & 1) ? N / 2 + (k >> 1) : k >> 1; }
template <int N>
__device__ __forceinline__ int tr_entry(int j) { return j < N / 2 ? 2 * j : 2 * (j - N / 2) + 1; }

// Output rows of the transpose owned by thread t: i = 4 g + u, a = t + g T,
// rows {a, P - a, P + a, N - a} all unpack from the same pair (Z_a, Z_{P-a}),
// so every Z is read once. a = 0 pairs rows {0, P} (Z_0) with {P/2, 3P/2}
// (Z_{P/2}), i.e. u = 1, 3 use a1 = P/2.
template <int N>
__device__ __forceinline__ int tr_row(int t, int i) {
  constexpr int P = N / 2, T = N / 16;
  const int u = i & 3, a = t + (i >> 2) * T, a1 = a ? a : P / 2;
  return u == 0 ? a : u == 1 ? P - a1 : u == 2 ? P + a : N - a1;
}

// X_kk of DCT-II row kk from V = (Za + conj Zb)/2 + e^{-2 pi i kk/N} (Za - conj Zb)/(2i),
// X = Re(conj(h) V), h = e^{i pi kk/(2N)}; tn = e^{i pi n/(2N)}, rn = e^{2 pi i n/N}
// of the output row n (kk = n, or N - n for the DST^T of odd terms).
template <bool ODD>
// (Returns 2 X: the 1/2 of V is applied by the caller, with the term's sign.)
__device__ __forceinline__ double tr_unpack(double2 za, double2 zc, double2 tn, double2 rn) {
  const double2 ev = make_double2(za.x + zc.x, za.y - zc.y);
  const double2 od = make_double2(za.y + zc.y, zc.x - za.x);
  const double2 r = ODD ? rn : make_double2(rn.x, -rn.y);
  const double2 h = ODD ? make_double2(tn.y, tn.x) : tn;
  const double2 Vv = make_double2(ev.x + od.x * r.x - od.y * r.y, ev.y + od.x * r.y + od.y * r.x);
  return h.x * Vv.x + h.y * Vv.y;
}

// One transposed term: o[i] += sign rp[i] X_{tr_row(t, i)}. The pack reads
// every stage entry exactly once. PM = 0: the stage as is; PM = 1 (Taylor):
// it also writes the next term's stage, h (N delta)/(l+1) = h * nd * inv_next
// (nd in the tr_slot order), into `next`; PM = 2 (Chebyshev): the stage is
// the input g and each entry is weighted on the fly by wrow[slot] (the
// term's weights in the tr_slot order). The first pass stores into zx;
// ping-pong (C::PP) as in fwd_term (returns the buffer the unpack read; the
// caller passes the other one as the next zx), else in place with a barrier
// ordering the first store after the previous term's unpack reads.
// TMO: the 16 output accumulators live in the thread's TMEM lane at tO
// (loaded, updated and stored back per row group) instead of o[].
// HST: the stage is the thread's own 16 pack entries in its TMEM lane at tH
// (r-major pairs), not hs.
template <int LOG2N, bool ODD, int PM, bool PPX = Cfg<LOG2N>::PP, int PST = 1, bool TMO = false,
          bool HST = false>
__device__ __forceinline__ double2* tr_term(const double* hs, double* next, const double* nd,
                                            const double* __restrict__ delta, double inv_next,
                                            const double* __restrict__ wrow, double2* zx,
                                            double2* zy, int t, int bar, double2 ta_t,
                                            double2 r4_t, const double2* fftw, const double* rp,
                                            double* o, double sign, uint32_t tO = 0,
                                            uint32_t tH = 0) {
  using C = Cfg<LOG2N>;
  constexpr int N = C::N, P = C::P, T = C::T, E = C::E, OWN = C::OWN;
  static_assert(E == 8 && T == N / 16, "row grouping assumes T = N/16");
  // pack v_q = h_{2q} (q < P), v_{N-1-q} = h_{2q+1}; z_m = v_{2m} + i v_{2m+1};
  // odd terms (DST^T) use (-1)^k h_k, i.e. negate the odd-index entries.
  // m < N/4: (h_{4m}, h_{4m+2}) = hs[2m .. 2m+1]; else (h_{2(N-1-2m)+1}, h_{2(N-2-2m)+1})
  // = the swapped pair at hs[P + N - 2 - 2m].
  double2 v[E];
  uint32_t hw[HST ? 16 : 1];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int m = t + r * T;
    const int slot = r < 4 ? 2 * m : P + N - 2 - 2 * m;
    double2 w;
    if constexpr (HST) {
      if (r == 0 || r == 4) {
        tm_ld8_nw(tH + 4 * r, hw);
        tm_ld8_nw(tH + 4 * r + 8, hw + 8);
        tm_wait_ld();
      }
      w = make_double2(join2(&hw[4 * (r & 3)]), join2(&hw[4 * (r & 3) + 2]));
    } else {
      w = *reinterpret_cast<const double2*>(hs + slot);
    }
    if (PM == 2) {
      const double2 q = __ldg(reinterpret_cast<const double2*>(wrow + slot));
      w = make_double2(w.x * q.x, w.y * q.y);
    }
    if (PM == 1) {
      const double2 q = C::SMEM_TABLES  // PM = 1 (Taylor) kernels use the Cfg layout
                            ? *reinterpret_cast<const double2*>(nd + slot)
                            : make_double2((double)N * __ldg(&delta[tr_entry<N>(slot)]),
                                           (double)N * __ldg(&delta[tr_entry<N>(slot + 1)]));
      *reinterpret_cast<double2*>(next + slot) = make_double2(w.x * (q.x * inv_next), w.y * (q.y * inv_next));
    }
    if (r < 4)
      v[r] = w;
    else
      v[r] = ODD ? make_double2(-w.y, -w.x) : make_double2(w.y, w.x);
  }
  pass_compute<P, E, 8, 1, false>(v, t, fftw);
  double2* zb = zx;
  if constexpr (PPX) {
    pass_store<P, E, 8, 1>(v, zx, t);
    group_sync<C::GT>(bar);
    zb = mid_passes_pp<P, E, 8, P, false, C::GT>(zx, zy, t, fftw, bar);
  } else {
    group_sync<C::GT>(bar);
    pass_store<P, E, 8, 1>(v, zx, t);
    group_sync<C::GT>(bar);
    mid_passes<P, E, 8, P, false, C::GT>(zx, t, fftw, bar);  // TWP measured slower here
  }
  constexpr double h = 0.70710678118654752440;
#pragma unroll
  for (int g = 0; g < OWN / 4; ++g) {
    const int a = t + g * T;
    // A = e^{i pi a/(2N)} = ta_t c32[g], R = e^{2 pi i a/N} = r4_t c8[g]
    const double2 A = make_double2(ta_t.x * kC32[g][0] - ta_t.y * kC32[g][1],
                                   ta_t.x * kC32[g][1] + ta_t.y * kC32[g][0]);
    const double2 R = make_double2(r4_t.x * kC8[g][0] - r4_t.y * kC8[g][1],
                                   r4_t.x * kC8[g][1] + r4_t.y * kC8[g][0]);
    const double2 zA = zb[smem_pad(a)], zB = zb[smem_pad((P - a) & (P - 1))];
    double2 A1 = A, R1 = R, zA1 = zA, zB1 = zB;
    if (a == 0) {  // rows P/2, 3P/2: a1 = P/2
      A1 = make_double2(kC32[4][0], kC32[4][1]);  // e^{i pi/8}
      R1 = make_double2(0.0, 1.0);
      zA1 = zB1 = zb[smem_pad(P / 2)];
    }
    // e^{i pi n/(2N)}, e^{2 pi i n/N} of the four rows, by symmetry from A, R
    const double2 t0 = A, r0 = R;                                                      // n = a
    const double2 t1 = make_double2(h * (A1.x + A1.y), h * (A1.x - A1.y));             // P - a1
    const double2 r1 = make_double2(-R1.x, R1.y);
    const double2 t2 = make_double2(h * (A.x - A.y), h * (A.x + A.y));                 // P + a
    const double2 r2 = make_double2(-R.x, -R.y);
    const double2 t3 = make_double2(A1.y, A1.x);                                       // N - a1
    const double2 r3 = make_double2(R1.x, -R1.y);
    // (Z_{kk mod P}, Z_{(P - kk) mod P}) of each row; the DST^T (kk = N - n) swaps them
    const double x0 = ODD ? (a == 0 ? 0.0 : tr_unpack<true>(zB, zA, t0, r0)) : tr_unpack<false>(zA, zB, t0, r0);
    const double x1 = ODD ? tr_unpack<true>(zA1, zB1, t1, r1) : tr_unpack<false>(zB1, zA1, t1, r1);
    const double x2 = ODD ? tr_unpack<true>(zB, zA, t2, r2) : tr_unpack<false>(zA, zB, t2, r2);
    const double x3 = ODD ? tr_unpack<true>(zA1, zB1, t3, r3) : tr_unpack<false>(zB1, zA1, t3, r3);
    // x_j = 2 X (tr_unpack): the 1/2 rides on the sign (exact)
    const double hs2 = 0.5 * sign;
    if constexpr (TMO) {
      uint32_t ow[8];
      tm_ld8(tO + 8 * g, ow);
      split2(join2(&ow[0]) + hs2 * (PST == 1 ? rp[4 * g + 0] : __ldg(rp + (4 * g + 0) * PST)) * x0, &ow[0]);
      split2(join2(&ow[2]) + hs2 * (PST == 1 ? rp[4 * g + 1] : __ldg(rp + (4 * g + 1) * PST)) * x1, &ow[2]);
      split2(join2(&ow[4]) + hs2 * (PST == 1 ? rp[4 * g + 2] : __ldg(rp + (4 * g + 2) * PST)) * x2, &ow[4]);
      split2(join2(&ow[6]) + hs2 * (PST == 1 ? rp[4 * g + 3] : __ldg(rp + (4 * g + 3) * PST)) * x3, &ow[6]);
      tm_st8(tO + 8 * g, ow);
    } else {
      o[4 * g + 0] += hs2 * (PST == 1 ? rp[4 * g + 0] : __ldg(rp + (4 * g + 0) * PST)) * x0;
      o[4 * g + 1] += hs2 * (PST == 1 ? rp[4 * g + 1] : __ldg(rp + (4 * g + 1) * PST)) * x1;
      o[4 * g + 2] += hs2 * (PST == 1 ? rp[4 * g + 2] : __ldg(rp + (4 * g + 2) * PST)) * x2;
      o[4 * g + 3] += hs2 * (PST == 1 ? rp[4 * g + 3] : __ldg(rp + (4 * g + 3) * PST)) * x3;
    }
  }
  if constexpr (TMO) tm_wait_st();
  return zb;
}

// BES: Chebyshev (Jacobi-Anger) expansion: the stage is the (weighted) input
// itself, each term weights it on the fly from wtab[m][slot] (tr_slot order)
// and scales the output rows by ttab[m][i T + t] = T_m(n/N) (tr_row order).
template <int LOG2N, bool BES>
__global__ void __launch_bounds__(Cfg<LOG2N>::THREADS, TrCfg<LOG2N, BES>::MINB)
    fast_ndct_tr_kernel(const double* __restrict__ in, size_t ld_in, double* __restrict__ out,
                        size_t ld_out, size_t batch, const double* __restrict__ delta,
                        int num_terms, int plain_op, const double* __restrict__ mult,
                        const double2* __restrict__ tw4n, const double2* __restrict__ fftw_g,
                        const double* __restrict__ wtab, const double* __restrict__ ttab,
                        int* nonfinite, int swap) {
  using C = Cfg<LOG2N>;
  using TC = TrCfg<LOG2N, BES>;
  constexpr int N = C::N, T = C::T, OWN = C::OWN;
  extern __shared__ double smem[];
  double* nd = smem + C::COLS * (TC::COL_BYTES / 8);
  double2* fftw_s = reinterpret_cast<double2*>(nd + N);
  const double2* fftw = TC::TABLES ? fftw_s : fftw_g;
  if (TC::TABLES) {
    if (plain_op < 0 && !BES)  // in the tr_slot layout of the stage
      for (int j = threadIdx.x; j < N; j += blockDim.x) nd[j] = (double)N * delta[tr_entry<N>(j)];
    load_table(fftw_s, fftw_g, C::TW);
    __syncthreads();
  }
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int bar = 1 + g;
  const size_t col = (size_t)blockIdx.x * C::COLS + g;
  if (col >= batch) return;
  // h_k = (N delta_k)^l / l! g_k at hs[tr_slot(k)], double-buffered by term parity
  double* hs = smem + g * (TC::COL_BYTES / 8);  // (not used with T3)
  double* hs_odd = hs + N;  // (Taylor only)
  double2* zbA = reinterpret_cast<double2*>(hs + (TC::T3 ? 0 : TC::ONE_STAGE ? 1 : 2) * N);
  double2* zbB = TC::PP ? zbA + C::ZB / sizeof(double2) : zbA;
  double2* zx = zbA;  // the first pass's target this term
  auto other = [&](double2* b) { return b == zbA ? zbB : zbA; };
  const double* src = in + col * ld_in;
  double o[OWN], rp[OWN];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < OWN; ++i) {
    o[i] = 0.0;
    rp[i] = 1.0;
  }
  if constexpr (!TC::T3) {
#pragma unroll
    for (int i = 0; i < OWN; ++i) {
      const int k = t + T * i;
      double v = src[k];
      if (mult) v = mult[k] * v;  // transforms.hpp:59 weighted = w_k f_k
      bad |= !isfinite(v);
      hs[tr_slot<N>(k)] = v;
    }
    if (bad && nonfinite) atomicOr(nonfinite, 1);
  }
  const double2 ta_t = __ldg(&tw4n[t]);      // e^{i pi t/(2N)}
  const double2 r4_t = __ldg(&tw4n[4 * t]);  // e^{2 pi i t/N}
  group_sync<C::GT>(bar);
  if (plain_op >= 0) {
    if (plain_op == 1)
      tr_term<LOG2N, true, 0, TC::PP>(hs, nullptr, nd, delta, 0.0, nullptr, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                              rp, o, 1.0);
    else
      tr_term<LOG2N, false, 0, TC::PP>(hs, nullptr, nd, delta, 0.0, nullptr, zx, other(zx), t, bar, ta_t, r4_t, fftw,
                               rp, o, 1.0);
  } else if (BES && TC::TMO) {
    // as below, with the output accumulators in TMEM (TrCfg::TMO)
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base))),
                   "n"(kTrCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tO = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) +
                        (uint32_t)(kTrCols / 2) * (uint32_t)(warp >> 2);
    const uint32_t tH = tO + 32;  // (T3) the thread's 16 pack entries
    {
      uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int q = 0; q < 4; ++q) tm_st8(tO + 8 * q, z);
      if constexpr (TC::T3) {
        // the entries (k0, k1) of pack slot pair r: (4m, 4m + 2) for r < 4, the
        // odd pair (2N - 3 - 4m, 2N - 1 - 4m) for r >= 4 (m = t + r T)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t hw8[8];
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int r = 2 * q + rr, m = t + r * T;
            const int k0 = r < 4 ? 4 * m : 2 * N - 3 - 4 * m, k1 = k0 + 2;
            double v0 = src[k0], v1 = src[k1];
            if (mult) {
              v0 *= mult[k0];
              v1 *= mult[k1];
            }
            bad |= !isfinite(v0) || !isfinite(v1);
            split2(v0, &hw8[4 * rr]);
            split2(v1, &hw8[4 * rr + 2]);
          }
          tm_st8(tH + 8 * q, hw8);
        }
        if (bad && nonfinite) atomicOr(nonfinite, 1);
      }
      tm_wait_st();
    }
    for (int m = 0; m < num_terms; ++m) {
      const double* tr = ttab + (size_t)m * N + t;
      const double* wrow = wtab + (size_t)m * N;
      double2* fin;
      if ((m & 1) ^ swap)
        fin = tr_term<LOG2N, true, 2, true, T, true, TC::T3>(hs, nullptr, nd, delta, 0.0, wrow, zx,
                                                             other(zx), t, bar, ta_t, r4_t, fftw, tr,
                                                             o, 1.0, tO, tH);
      else
        fin = tr_term<LOG2N, false, 2, true, T, true, TC::T3>(hs, nullptr, nd, delta, 0.0, wrow, zx,
                                                              other(zx), t, bar, ta_t, r4_t, fftw, tr,
                                                              o, 1.0, tO, tH);
      zx = other(fin);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t ow[8];
      tm_ld8(tO + 8 * q, ow);
#pragma unroll
      for (int j = 0; j < 4; ++j) o[4 * q + j] = join2(&ow[2 * j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(kTrCols)
                   : "memory");
  } else if (BES && TC::TWO) {
    // row factors read where they are applied (PST = T): fewer live registers;
    // ping-pong rows when the second stage buffer is free (ONE_STAGE)
    for (int m = 0; m < num_terms; ++m) {
      const double* tr = ttab + (size_t)m * N + t;
      const double* wrow = wtab + (size_t)m * N;
      double2* fin;
      if ((m & 1) ^ swap)
        fin = tr_term<LOG2N, true, 2, TC::ONE_STAGE, T>(hs, nullptr, nd, delta, 0.0, wrow, zx,
                                                       other(zx), t, bar, ta_t, r4_t, fftw, tr, o, 1.0);
      else
        fin = tr_term<LOG2N, false, 2, TC::ONE_STAGE, T>(hs, nullptr, nd, delta, 0.0, wrow, zx,
                                                        other(zx), t, bar, ta_t, r4_t, fftw, tr, o, 1.0);
      if (TC::ONE_STAGE) zx = other(fin);
    }
  } else if (BES) {
    for (int m = 0; m < num_terms; ++m) {
#pragma unroll
      for (int i = 0; i < OWN; ++i) rp[i] = __ldg(ttab + (size_t)m * N + i * T + t);
      const double* wrow = wtab + (size_t)m * N;
      double2* fin;
      if ((m & 1) ^ swap)
        fin = tr_term<LOG2N, true, 2, TC::PP>(hs, nullptr, nd, delta, 0.0, wrow, zx, other(zx), t, bar,
                                      ta_t, r4_t, fftw, rp, o, 1.0);
      else
        fin = tr_term<LOG2N, false, 2, TC::PP>(hs, nullptr, nd, delta, 0.0, wrow, zx, other(zx), t, bar,
                                       ta_t, r4_t, fftw, rp, o, 1.0);
      zx = other(fin);
    }
  } else {
    for (int l = 0; l < num_terms; ++l) {
      if (l > 0) {
#pragma unroll
        for (int i = 0; i < OWN; ++i)
          rp[i] *= (double)tr_row<N>(t, i) / (double)N;  // (n/N)^l for output row n
      }
      const double inv_next = 1.0 / (double)(l + 1);
      double2* fin;
      if (l & 1)
        fin = tr_term<LOG2N, true, 1, TC::PP>(hs_odd, hs, nd, delta, inv_next, nullptr, zx, other(zx), t,
                                      bar, ta_t, r4_t, fftw, rp, o, taylor_sign_d(l));
      else
        fin = tr_term<LOG2N, false, 1, TC::PP>(hs, hs_odd, nd, delta, inv_next, nullptr, zx, other(zx), t,
                                       bar, ta_t, r4_t, fftw, rp, o, taylor_sign_d(l));
      zx = other(fin);
    }
  }
  double* dst = out + col * ld_out;
#pragma unroll
  for (int i = 0; i < OWN; ++i) dst[tr_row<N>(t, i)] = o[i];
}

// One plain DCT-III / DST-III (odd = 1) or transpose per column: the
// trig.hpp passes on the cheb1 grid. A single term needs neither the stage
// double buffer nor ping-pong FFT rows nor shared tables, so a CTA takes
// N*8 + one FFT row of shared memory and <= 128 registers: two or three CTAs
// per SM overlap one column's loads with another's FFT (the pass is HBM-bound,
// the many-term kernels above are not).
template <int LOG2N>
__global__ void __launch_bounds__(Cfg<LOG2N>::THREADS, 2)
    fast_dct_plain_fwd_kernel(const double* __restrict__ in, size_t ld_in, double* __restrict__ out,
                              size_t ld_out, size_t batch, int odd,
                              const double2* __restrict__ tw4n, const double2* __restrict__ fftw,
                              int* nonfinite) {
  using C = Cfg<LOG2N>;
  constexpr int N = C::N, T = C::T, OWN = C::OWN;
  constexpr size_t COLW = N + C::ZB / sizeof(double);
  extern __shared__ double smem[];
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int bar = 1 + g;
  const size_t col = (size_t)blockIdx.x * C::COLS + g;
  if (col >= batch) return;
  double* stage = smem + g * COLW;
  double2* zb = reinterpret_cast<double2*>(stage + N);
  const double* src = in + col * ld_in;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < OWN; ++i) {
    const double v = __ldcs(src + t + T * i);
    bad |= !isfinite(v);
    stage[t + T * i] = v;
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
  double f[OWN], p[OWN];
#pragma unroll
  for (int i = 0; i < OWN; ++i) {
    f[i] = 0.0;
    p[i] = 1.0;
  }
  const double2 ta_t = __ldg(&tw4n[t]);
  const double2 r4_t = __ldg(&tw4n[4 * t]);
  group_sync<C::GT>(bar);
  if (odd)
    fwd_term<LOG2N, true, 0, false>(stage, nullptr, zb, zb, t, bar, ta_t, r4_t, fftw, p, f, 1.0);
  else
    fwd_term<LOG2N, false, 0, false>(stage, nullptr, zb, zb, t, bar, ta_t, r4_t, fftw, p, f, 1.0);
  group_sync<C::GT>(bar);
#pragma unroll
  for (int i = 0; i < OWN; ++i) stage[out_slot(fwd_own_row<LOG2N>(t, i))] = f[i];
  group_sync<C::GT>(bar);
  double* dst = out + col * ld_out;
#pragma unroll
  for (int i = 0; i < OWN; ++i) __stcs(dst + t + T * i, stage[out_slot(t + T * i)]);
}

// Persistent, prefetching variant of the plain forward pass for one column
// per CTA (N >= 4096): while a CTA transforms column i, a bulk copy
// (cp.async.bulk, mbarrier completion) brings column i + grid into the other
// stage buffer, so the column load no longer stalls the FFT.
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_init1(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra D_%=;\n\t"
      "bra W_%=;\n"
      "D_%=:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Shared memory: one stage buffer, one FFT row, the pass twiddles. The next
// column's bulk copy into the stage buffer is issued as soon as every thread
// has packed the current one (after the first pass's barrier), so it overlaps
// the remaining passes; the output is staged through the FFT row.
// Twiddles in shared memory at two CTAs per SM (1.30 ms for 65536 columns of
// 4096) beat global twiddles at three CTAs and 80 registers (1.43 ms, spills).
#ifndef FLB_STREAM_TW_SMEM
#define FLB_STREAM_TW_SMEM 1
#endif
#ifndef FLB_STREAM_PP
#define FLB_STREAM_PP 1
#endif
template <int LOG2N>
struct StreamCfg {
  using C = Cfg<LOG2N>;
  // outputs straight from the mirrored radix-4 last pass (no staging)
  static constexpr bool DIRECT_OUT = C::RL == 4 && C::E / C::RL == 2;
  // PP: two FFT rows used alternately per column and per pass (ping-pong):
  // one barrier per pass and none between columns; the twiddles then stay
  // in global memory (L1) so that two CTAs still fit per SM
  static constexpr bool PP = FLB_STREAM_PP && DIRECT_OUT && LOG2N <= 12;
  static constexpr bool TW_SMEM = FLB_STREAM_TW_SMEM != 0 && !PP;
  static constexpr size_t SMEM = C::N * sizeof(double) + (PP ? 2 : 1) * C::ZB +
                                 (TW_SMEM ? C::TW * sizeof(double2) : 0);
  static constexpr int MINB = LOG2N <= 12 ? (TW_SMEM || PP ? 2 : 3) : 1;
};

template <int LOG2N>
__global__ void __launch_bounds__(Cfg<LOG2N>::THREADS, StreamCfg<LOG2N>::MINB)
    fast_dct_stream_fwd_kernel(const double* __restrict__ in, size_t ld_in,
                               double* __restrict__ out, size_t ld_out, size_t batch, int odd,
                               const double2* __restrict__ tw4n, const double2* __restrict__ fftw_g,
                               int* nonfinite) {
  using C = Cfg<LOG2N>;
  static_assert(C::COLS == 1, "one column per CTA");
  constexpr int N = C::N, P = C::P, T = C::T, E = C::E, OWN = C::OWN, NSL = C::NSL, RL = C::RL;
  extern __shared__ double smem[];
  __shared__ uint64_t mbar;
  double* stage = smem;
  double2* zb = reinterpret_cast<double2*>(smem + N);
  double* zo = smem + N;  // output staging (the FFT row, after the last pass)
  double2* fftw_s = reinterpret_cast<double2*>(smem + N + C::ZB / sizeof(double));
  const double2* fftw = StreamCfg<LOG2N>::TW_SMEM ? fftw_s : fftw_g;
  // radix-4 last pass, two butterflies per thread: outputs go straight out
  constexpr bool DIRECT_OUT = StreamCfg<LOG2N>::DIRECT_OUT;
  constexpr bool PP = StreamCfg<LOG2N>::PP;
  double2* zb2 = zb + C::ZB / sizeof(double2);  // PP: the second FFT row
  const int t = threadIdx.x;
  const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar));
  const uint32_t stage_s = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
  if (t == 0) {
    mbar_init1(bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (StreamCfg<LOG2N>::TW_SMEM) load_table(fftw_s, fftw_g, C::TW);
  __syncthreads();
  size_t col = blockIdx.x;
  if (t == 0 && col < batch) {
    mbar_expect(bar, N * 8);
    bulk_load(stage_s, in + col * ld_in, N * 8, bar);
  }
  const double2 ta_t = __ldg(&tw4n[t]);
  const double2 r4_t = __ldg(&tw4n[4 * t]);
  bool bad = false;
  for (uint32_t it = 0; col < batch; col += gridDim.x, ++it) {
    // PP: this column's first pass writes the row the previous column's last
    // pass did not read, and every later pass sits behind a CTA barrier that
    // all of the previous column's reads precede
    double2* za = PP && (it & 1u) ? zb2 : zb;
    double2* zo2 = PP && (it & 1u) ? zb : zb2;
    if constexpr (!PP) __syncthreads();  // the previous column's output has left the FFT row
    mbar_wait_parity(bar, it & 1u);
    double2 v[E];
    if (odd)
      fwd_pack_all<N, true, 0, 0>(v, stage, nullptr, t, ta_t, r4_t, &bad);
    else
      fwd_pack_all<N, false, 0, 0>(v, stage, nullptr, t, ta_t, r4_t, &bad);
    pass_compute<P, E, 8, 1, true>(v, t, fftw);
    pass_store<P, E, 8, 1>(v, za, t);
    __syncthreads();  // every thread has packed: the stage buffer takes the next column
    const size_t nxt = col + gridDim.x;
    if (t == 0 && nxt < batch) {
      mbar_expect(bar, N * 8);
      bulk_load(stage_s, in + nxt * ld_in, N * 8, bar);
    }
    double2* fin = za;
    if constexpr (PP)
      fin = mid_passes_pp<P, E, 8, NSL, true, 0, true>(za, zo2, t, fftw, 0);
    else
      mid_passes<P, E, 8, NSL, true, 0, true>(zb, t, fftw, 0);
    double* dst = out + col * ld_out;
    if constexpr (DIRECT_OUT) {
      // mirrored last-pass butterflies: z_m (rows 4m, 4m + 2) and z_{P-1-m}
      // (rows 4m + 3, 4m + 1) in one thread = four contiguous output rows,
      // stored straight from registers (no staging, two barriers fewer)
      pass_load<P, E, RL, true>(v, fin, t);
      pass_compute<P, E, RL, NSL, true, true, true>(v, t, fftw + pass_tw_offset(P, NSL));
      // A warp's 32 blocks of one r are 1 KB contiguous (ascending in the
      // lane for m < P/2, descending above); two lane shuffles per half let
      // each 16-byte store instruction cover 512 contiguous bytes.
      const double sg = odd ? -1.0 : 1.0;  // DST: odd rows negated
      const int lane = t & 31, wbase = t - lane;
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        const int m = t + r * NSL;
        const double2 a = v[r], b = v[RL + RL - 1 - r];  // z_m, z_{P-1-m}
        const bool lo = r * NSL < P / 2;                  // (warp-uniform)
        const double2 z = lo ? a : b, w = lo ? b : a;     // z: rows 4m', 4m' + 2
        const double2 h0 = make_double2(z.x, sg * w.y), h1 = make_double2(z.y, sg * w.x);
        // the warp's lowest block: lane 0 (ascending) or lane 31 (descending)
        const int blk0 = lo ? wbase + r * NSL : P - 1 - (wbase + 31 + r * NSL);
        (void)m;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int bi = 16 * hh + (lane >> 1);  // block in address order
          const int src = lo ? bi : 31 - bi;
          double2 g0, g1;
          g0.x = __shfl_sync(0xffffffffu, h0.x, src);
          g0.y = __shfl_sync(0xffffffffu, h0.y, src);
          g1.x = __shfl_sync(0xffffffffu, h1.x, src);
          g1.y = __shfl_sync(0xffffffffu, h1.y, src);
          __stcs(reinterpret_cast<double2*>(dst + 4 * blk0 + 64 * hh + 2 * lane),
                 (lane & 1) ? g1 : g0);
        }
      }
    } else {
      pass_load<P, E, RL>(v, zb, t);
      pass_compute<P, E, RL, NSL, true, true>(v, t, fftw + pass_tw_offset(P, NSL));
      __syncthreads();  // all last-pass loads done: the FFT row stages the output
#pragma unroll
      for (int q = 0; q < E / RL; ++q)
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int m = t + q * T + r * NSL;
          const double2 z = v[q * RL + r];
          const int k0 = fwd_row_of<N>(2 * m), k1 = fwd_row_of<N>(2 * m + 1);
          zo[out_slot(k0)] = (odd && (k0 & 1)) ? -z.x : z.x;
          zo[out_slot(k1)] = (odd && (k1 & 1)) ? -z.y : z.y;
        }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < OWN; ++i) __stcs(dst + t + T * i, zo[out_slot(t + T * i)]);
    }
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
}

// Persistent, prefetching transposed pass (dct_iii_transpose /
// dst_iii_transpose, the DCT-II type) for one column per CTA (N >= 4096):
// the next column arrives by one contiguous bulk copy (cp.async.bulk,
// mbarrier completion) into the stage buffer as soon as every thread has
// packed the current one (after the first pass's barrier), so it overlaps
// the remaining passes. The pack reads its even/odd entry pairs straight
// from the natural-order column (no de-interleave copy, no element-strided
// global access), which leaves room for two FFT rows used alternately per
// pass and per column (ping-pong: one barrier per pass, none between
// columns) at two CTAs per SM.
template <int LOG2N>
__global__ void __launch_bounds__(Cfg<LOG2N>::THREADS, LOG2N <= 12 ? 2 : 1)
    fast_dct_stream_tr_kernel(const double* __restrict__ in, size_t ld_in,
                              double* __restrict__ out, size_t ld_out, size_t batch, int odd,
                              const double2* __restrict__ tw4n, const double2* __restrict__ fftw,
                              int* nonfinite) {
  using C = Cfg<LOG2N>;
  static_assert(C::COLS == 1, "one column per CTA");
  constexpr int N = C::N, P = C::P, T = C::T, E = C::E, OWN = C::OWN;
  extern __shared__ double smem[];
  __shared__ uint64_t mbar;
  double* raw = smem;  // the bulk-copied column, natural order
  double2* zbA = reinterpret_cast<double2*>(smem + N);
  double2* zbB = zbA + C::ZB / sizeof(double2);
  const int t = threadIdx.x;
  const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar));
  const uint32_t raw_s = static_cast<uint32_t>(__cvta_generic_to_shared(raw));
  if (t == 0) {
    mbar_init1(bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  size_t col = blockIdx.x;
  if (t == 0 && col < batch) {
    mbar_expect(bar, N * 8);
    bulk_load(raw_s, in + col * ld_in, N * 8, bar);
  }
  const double2 ta_t = __ldg(&tw4n[t]);
  const double2 r4_t = __ldg(&tw4n[4 * t]);
  bool bad = false;
  double2* zx = zbA;
  constexpr double h = 0.70710678118654752440;
#ifndef FLB_STREAM_TR_DEINTERLEAVE
#define FLB_STREAM_TR_DEINTERLEAVE 1
#endif
  for (uint32_t it = 0; col < batch; col += gridDim.x, ++it) {
    mbar_wait_parity(bar, it & 1u);
    double2* zy = zx == zbA ? zbB : zbA;
    double2 v[E];
    if constexpr (FLB_STREAM_TR_DEINTERLEAVE) {
      // de-interleave the column by parity into the free FFT row (even entries,
      // then odd ones): the pack's stride-4 reads of the natural-order column
      // were 4-way shared-memory bank conflicts (81.6 M per 65536 columns)
      double* ev = reinterpret_cast<double*>(zx);
      double* od = ev + N / 2;
#pragma unroll
      for (int r = 0; r < N / 2 / T; ++r) {
        const int i = t + r * T;
        const double2 w = *reinterpret_cast<const double2*>(raw + 2 * i);
        ev[i] = w.x;
        od[i] = w.y;
      }
      __syncthreads();  // the column is copied (and the previous unpack is done)
      const size_t nxt = col + gridDim.x;
      if (t == 0 && nxt < batch) {
        mbar_expect(bar, N * 8);
        bulk_load(raw_s, in + nxt * ld_in, N * 8, bar);
      }
      // pack (tr_term): v_r = (h_{4m}, h_{4m+2}) = ev[2m], ev[2m+1] for r < 4, the
      // swapped odd pair (h_{2N-3-4m}, h_{2N-1-4m}) = od[N-2-2m], od[N-1-2m]
      // for r >= 4 (m = t + r T); odd terms (DST^T) negate the odd-index entries
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const int m = t + r * T;
        const double2 w = r < 4 ? *reinterpret_cast<const double2*>(ev + 2 * m)
                                : *reinterpret_cast<const double2*>(od + (N - 2 - 2 * m));
        bad |= !isfinite(w.x) || !isfinite(w.y);
        v[r] = r < 4 ? w : (odd ? make_double2(-w.y, -w.x) : make_double2(w.y, w.x));
      }
      pass_compute<P, E, 8, 1, false>(v, t, fftw);
      pass_store<P, E, 8, 1>(v, zy, t);  // the other row (free after the barrier)
      __syncthreads();
    } else {
      // pack (tr_term) straight from the natural-order column
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const int m = t + r * T;
        const int k0 = r < 4 ? 4 * m : 2 * N - 3 - 4 * m;
        const double2 w = make_double2(raw[k0], raw[k0 + 2]);
        bad |= !isfinite(w.x) || !isfinite(w.y);
        v[r] = r < 4 ? w : (odd ? make_double2(-w.y, -w.x) : make_double2(w.y, w.x));
      }
      pass_compute<P, E, 8, 1, false>(v, t, fftw);
      pass_store<P, E, 8, 1>(v, zx, t);
      __syncthreads();  // every thread has packed: the stage buffer takes the next column
      const size_t nxt = col + gridDim.x;
      if (t == 0 && nxt < batch) {
        mbar_expect(bar, N * 8);
        bulk_load(raw_s, in + nxt * ld_in, N * 8, bar);
      }
      zy = zx;
      zx = zx == zbA ? zbB : zbA;
    }
    // zy holds the first pass; zx is free
#ifndef FLB_STREAM_TR_TWP
#define FLB_STREAM_TR_TWP 1  // 4096 x 65536: 1.108 -> 1.040 ms (59 -> 63 % of HBM)
#endif
    double2* zb = mid_passes_pp<P, E, 8, P, false, 0, FLB_STREAM_TR_TWP != 0>(zy, zx, t, fftw, 0);
    // unpack (tr_term): rows {a, P - a, P + a, N - a} of each group g
    double* dst = out + col * ld_out;
#pragma unroll
    for (int g = 0; g < OWN / 4; ++g) {
      const int a = t + g * T;
      const double2 A = make_double2(ta_t.x * kC32[g][0] - ta_t.y * kC32[g][1],
                                     ta_t.x * kC32[g][1] + ta_t.y * kC32[g][0]);
      const double2 R = make_double2(r4_t.x * kC8[g][0] - r4_t.y * kC8[g][1],
                                     r4_t.x * kC8[g][1] + r4_t.y * kC8[g][0]);
      const double2 zA = zb[smem_pad(a)], zB = zb[smem_pad((P - a) & (P - 1))];
      double2 A1 = A, R1 = R, zA1 = zA, zB1 = zB;
      if (a == 0) {
        A1 = make_double2(kC32[4][0], kC32[4][1]);
        R1 = make_double2(0.0, 1.0);
        zA1 = zB1 = zb[smem_pad(P / 2)];
      }
      const double2 t0 = A, r0 = R;
      const double2 t1 = make_double2(h * (A1.x + A1.y), h * (A1.x - A1.y));
      const double2 r1 = make_double2(-R1.x, R1.y);
      const double2 t2 = make_double2(h * (A.x - A.y), h * (A.x + A.y));
      const double2 r2 = make_double2(-R.x, -R.y);
      const double2 t3 = make_double2(A1.y, A1.x);
      const double2 r3 = make_double2(R1.x, -R1.y);
      double x0, x1, x2, x3;
      if (odd) {
        x0 = a == 0 ? 0.0 : tr_unpack<true>(zB, zA, t0, r0);
        x1 = tr_unpack<true>(zA1, zB1, t1, r1);
        x2 = tr_unpack<true>(zB, zA, t2, r2);
        x3 = tr_unpack<true>(zA1, zB1, t3, r3);
      } else {
        x0 = tr_unpack<false>(zA, zB, t0, r0);
        x1 = tr_unpack<false>(zB1, zA1, t1, r1);
        x2 = tr_unpack<false>(zA, zB, t2, r2);
        x3 = tr_unpack<false>(zB1, zA1, t3, r3);
      }
      const int a1 = a ? a : P / 2;
      __stcs(dst + a, 0.5 * x0);
      __stcs(dst + (P - a1), 0.5 * x1);
      __stcs(dst + (P + a), 0.5 * x2);
      __stcs(dst + (N - a1), 0.5 * x3);
    }
    zx = zb == zbA ? zbB : zbA;  // the next column's first pass: the row this unpack did not read
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
}

template <int LOG2N>
__global__ void __launch_bounds__(Cfg<LOG2N>::THREADS, 2)
    fast_dct_plain_tr_kernel(const double* __restrict__ in, size_t ld_in, double* __restrict__ out,
                             size_t ld_out, size_t batch, int odd,
                             const double2* __restrict__ tw4n, const double2* __restrict__ fftw,
                             int* nonfinite) {
  using C = Cfg<LOG2N>;
  constexpr int N = C::N, T = C::T, OWN = C::OWN;
  constexpr size_t COLW = N + C::ZB / sizeof(double);
  extern __shared__ double smem[];
  const int g = threadIdx.x / T, t = threadIdx.x % T;
  const int bar = 1 + g;
  const size_t col = (size_t)blockIdx.x * C::COLS + g;
  if (col >= batch) return;
  double* hs = smem + g * COLW;
  double2* zb = reinterpret_cast<double2*>(hs + N);
  const double* src = in + col * ld_in;
  double o[OWN], rp[OWN];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < OWN; ++i) {
    const int k = t + T * i;
    const double v = __ldcs(src + k);
    bad |= !isfinite(v);
    hs[tr_slot<N>(k)] = v;
    o[i] = 0.0;
    rp[i] = 1.0;
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
  const double2 ta_t = __ldg(&tw4n[t]);
  const double2 r4_t = __ldg(&tw4n[4 * t]);
  group_sync<C::GT>(bar);
  if (odd)
    tr_term<LOG2N, true, 0, false>(hs, nullptr, nullptr, nullptr, 0.0, nullptr, zb, zb, t, bar,
                                   ta_t, r4_t, fftw, rp, o, 1.0);
  else
    tr_term<LOG2N, false, 0, false>(hs, nullptr, nullptr, nullptr, 0.0, nullptr, zb, zb, t, bar,
                                    ta_t, r4_t, fftw, rp, o, 1.0);
  double* dst = out + col * ld_out;
#pragma unroll
  for (int i = 0; i < OWN; ++i) __stcs(dst + tr_row<N>(t, i), o[i]);
}

__global__ void tw4n_kernel(double2* tw, unsigned long long n) {
  const unsigned long long q = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (q >= 2 * n) return;
  double s, c;
  sincospi((double)q / (double)(2 * n), &s, &c);  // e^{2 pi i q / (4N)}
  tw[q] = make_double2(c, s);
}

const double2* tw4n_table(int log2n) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, double2*> tables;
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  double2*& slot = tables[{dev, log2n}];
  if (!slot) {
    const unsigned long long n = 1ull << log2n;
    FLB_CUDA(cudaMalloc(&slot, 2 * n * sizeof(double2)));
    tw4n_kernel<<<(unsigned)((2 * n + 255) / 256), 256>>>(slot, n);
    note_launch("tw4n_kernel");
    FLB_CUDA(cudaDeviceSynchronize());
  }
  return slot;
}

template <int LOG2N>
void launch_fast(int transpose, const double* in, size_t ld_in, double* out, size_t ld_out,
                 size_t batch, const double* delta, int num_terms, int plain_op,
                 const double* mult, int* nonfinite, cudaStream_t s, const FastNdct* bes) {
  using C = Cfg<LOG2N>;
  const double2* tw = tw4n_table(LOG2N);
  const double2* fftw = pass_twiddles(LOG2N - 1);
  const bool use_bes = bes && bes->bes_terms > 0 && plain_op < 0;
  const size_t max_cols = (size_t)0x7fffffff * C::COLS;
  if constexpr (C::COLS == 1) {
#ifndef FLB_STREAM_TR
#define FLB_STREAM_TR 1
#endif
    if (FLB_STREAM_TR && plain_op >= 0 && !mult && transpose && ld_in == ld_out &&
        (ld_in % 2) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
      const size_t smem = C::N * sizeof(double) + 2 * C::ZB;
      FLB_CUDA(cudaFuncSetAttribute(fast_dct_stream_tr_kernel<LOG2N>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const unsigned grid =
          (unsigned)std::min<size_t>(batch, (size_t)sm_count() * (LOG2N <= 12 ? 2 : 1));
      fast_dct_stream_tr_kernel<LOG2N><<<grid, C::THREADS, smem, s>>>(
          in, ld_in, out, ld_out, batch, plain_op, tw, fftw, nonfinite);
      note_launch("fast_dct_stream_tr_kernel");
      return;
    }
    if (plain_op >= 0 && !mult && !transpose && ld_in == ld_out && (ld_in % 2) == 0 &&
        (reinterpret_cast<uintptr_t>(in) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
      const size_t smem = StreamCfg<LOG2N>::SMEM;
      FLB_CUDA(cudaFuncSetAttribute(fast_dct_stream_fwd_kernel<LOG2N>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const unsigned grid =
          (unsigned)std::min<size_t>(batch, (size_t)sm_count() * StreamCfg<LOG2N>::MINB);
      fast_dct_stream_fwd_kernel<LOG2N><<<grid, C::THREADS, smem, s>>>(
          in, ld_in, out, ld_out, batch, plain_op, tw, fftw, nonfinite);
      note_launch("fast_dct_stream_fwd_kernel");
      return;
    }
  }
  if (plain_op >= 0 && !mult) {
    const size_t smem = C::COLS * (C::N * sizeof(double) + C::ZB);
    for (size_t c0 = 0; c0 < batch; c0 += max_cols) {
      const size_t nc = batch - c0 < max_cols ? batch - c0 : max_cols;
      const unsigned grid = (unsigned)((nc + C::COLS - 1) / C::COLS);
      auto kern = transpose ? fast_dct_plain_tr_kernel<LOG2N> : fast_dct_plain_fwd_kernel<LOG2N>;
      FLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<grid, C::THREADS, smem, s>>>(in + c0 * ld_in, ld_in, out + c0 * ld_out, ld_out, nc,
                                          plain_op, tw, fftw, nonfinite);
      note_launch(transpose ? "fast_dct_plain_tr_kernel" : "fast_dct_plain_fwd_kernel");
    }
    return;
  }
  for (size_t c0 = 0; c0 < batch; c0 += max_cols) {
    const size_t nc = batch - c0 < max_cols ? batch - c0 : max_cols;
    const unsigned grid = (unsigned)((nc + C::COLS - 1) / C::COLS);
    if (transpose) {
      auto kern = use_bes ? fast_ndct_tr_kernel<LOG2N, true> : fast_ndct_tr_kernel<LOG2N, false>;
      const int smem = use_bes ? (int)TrCfg<LOG2N, true>::SMEM : (int)TrCfg<LOG2N, false>::SMEM;
      FLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<grid, C::THREADS, smem, s>>>(
          in + c0 * ld_in, ld_in, out + c0 * ld_out, ld_out, nc, delta,
          use_bes ? bes->bes_terms : num_terms, plain_op, mult, tw, fftw,
          use_bes ? bes->bes_wt : nullptr, use_bes ? bes->bes_tt : nullptr, nonfinite,
          use_bes ? bes->swap : 0);
      note_launch(use_bes ? "fast_ndct_tr_kernel<bessel>" : "fast_ndct_tr_kernel");
    } else {
      auto kern = use_bes ? fast_ndct_fwd_kernel<LOG2N, true> : fast_ndct_fwd_kernel<LOG2N, false>;
      const int smem = use_bes ? (int)FwdCfg<LOG2N, true>::SMEM : (int)FwdCfg<LOG2N, false>::SMEM;
      FLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<grid, C::THREADS, smem, s>>>(
          in + c0 * ld_in, ld_in, out + c0 * ld_out, ld_out, nc, delta,
          use_bes ? bes->bes_terms : num_terms, plain_op, tw, fftw,
          use_bes ? bes->bes_wf : nullptr, nonfinite, use_bes ? bes->swap : 0);
      note_launch(use_bes ? "fast_ndct_fwd_kernel<bessel>" : "fast_ndct_fwd_kernel");
    }
  }
}

// J_m(y), |y| <~ 1, by its power series (alternating, decreasing terms).
__host__ __device__ inline double bessel_j(int m, double y) {
  const double h = 0.5 * y;
  double t = 1.0;
  for (int i = 1; i <= m; ++i) t *= h / (double)i;
  double sum = t;
  for (int k = 1; k < 40; ++k) {
    t *= -(h * h) / ((double)k * (double)(m + k));
    sum += t;
    if (fabs(t) <= 1e-18 * fabs(sum)) break;
  }
  return sum;
}

// Weight of term m (sign and Jacobi-Anger factor included):
//   cos(x y) = J_0 + 2 sum_k (-1)^k J_2k(y) T_2k(x),  sin(x y) = 2 sum_k (-1)^k J_2k+1(y) T_2k+1(x),
//   cos(n theta_k) = cos(n theta0_k) cos(x y) - sin(n theta0_k) sin(x y), x = n/N, y = N delta_k.
__host__ __device__ inline double bessel_weight(int m, double y) {
  const double j = bessel_j(m, y);
  if ((m & 1) == 0) return (m == 0 ? 1.0 : 2.0) * (((m >> 1) & 1) ? -j : j);
  return -2.0 * ((((m - 1) >> 1) & 1) ? -j : j);
}

// ---------------------------------------------------------------------------
// 8192 < N <= 2^16: the forward Chebyshev-expansion NDCT of one column fused
// on a thread-block CLUSTER, all terms on chip. The N/2-point
// complex FFT of each term is a four-step over CS = N/8192 CTAs:
//   P = CS Q (Q = 4096), m = CS m2 + m1 (CTA m1 packs Z at its m2 = t + T r),
//   Y_{m1}[k1] = sum_{m2} Z_{CS m2 + m1} w_Q^{m2 k1}      (local smem FFT)
//   z_{k1 + Q k2} = sum_{m1} (w_P^{m1 k1} Y_{m1}[k1]) w_CS^{m1 k2}
//                                     (CTA s: k1 in [s Q/CS, (s+1) Q/CS), the
//                                      Y rows of all CTAs read through DSMEM)
// (inverse transforms, w = e^{+2 pi i/.}). The stage T_m(n/N) c lives in the
// CTAs' shared memory (entry n = CS a + m1 at st[a]); the pack's mirror
// entries N - m, P - m sit in CTA (CS - m1) mod CS and are read through DSMEM;
// the previous stage stays in registers; the 16 outputs a thread's z values
// map to accumulate in registers over all terms with weights from a table in
// thread order (signs folded in). Two cluster barriers per term: Y rows
// complete (and every pack done, so the stage may be updated), and every
// Y read / stage write done before the next term. c is read once, f written
// once; the Z / Y traffic stays in shared memory (~94 % of it local).
template <int LOG2N>
struct ClCfg {
  static constexpr int N = 1 << LOG2N, P = N / 2;
  static constexpr int Q = 4096;          // local FFT points per CTA
  static constexpr int CS = P / Q;        // CTAs per column
  static constexpr int T = 512, E = 8;    // threads, local points per thread
  static constexpr int KQ = Q / CS;       // step-C k1 per CTA
  static constexpr int D = KQ / T;        // k1 per thread
  static constexpr int OUTS = 2 * D * CS;  // outputs per thread (16)
  // the stage, the previous stage (own entries only), the FFT row
  static constexpr size_t SMEM = (size_t)4 * Q * sizeof(double) + (size_t)smem_row(Q) * sizeof(double2);
  static_assert(CS >= 2 && CS <= 8 && KQ % T == 0 && OUTS == 16, "2^14 <= N <= 2^16");
};

// Output row of slot i (= 2 (d CS + k2) + part) of thread t in CTA s.
template <int LOG2N>
__host__ __device__ __forceinline__ int cl_out_row(int s, int t, int i) {
  using C = ClCfg<LOG2N>;
  const int part = i & 1, zi = i >> 1, d = zi / C::CS, k2 = zi % C::CS;
  const int k = s * C::KQ + t + d * C::T + C::Q * k2;  // z index
  const int q = 2 * k + part;
  return q < C::N / 2 ? 2 * q : 2 * (C::N - 1 - q) + 1;
}

template <int LOG2N>
__global__ void __launch_bounds__(512, 1)
    cluster_ndct_fwd_kernel(const double* __restrict__ in, size_t ld_in, double* __restrict__ out,
                            size_t ld_out, int terms, int swap, const double* __restrict__ wt,
                            const double2* __restrict__ tw4n, const double2* __restrict__ fftw,
                            int* nonfinite) {
  namespace cg = cooperative_groups;
  using C = ClCfg<LOG2N>;
  constexpr int N = C::N, Q = C::Q, CS = C::CS, T = C::T, E = C::E, KQ = C::KQ, D = C::D;
  extern __shared__ double smem[];
  double* st = smem;                                        // 2Q stage entries
  double* pv = smem + 2 * Q;                                // T_{m-1} c at the same entries
  double2* Y = reinterpret_cast<double2*>(smem + 4 * Q);   // the local FFT row
  cg::cluster_group cl = cg::this_cluster();
  const int m1 = (int)cl.block_rank();
  const size_t col = blockIdx.x / CS;
  const int t = threadIdx.x;
  const double* rst = cl.map_shared_rank(st, (CS - m1) % CS);  // the mirror CTA's stage
  const double* src = in + col * ld_in;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < E; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int a = h * Q + t + T * i;
      const double v = src[(size_t)CS * a + m1];
      bad |= !isfinite(v);
      st[a] = v;
    }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
  // step-C twiddle e^{+2 pi i r k1 / P} = e^{2 pi i (8 r k1) / (4N)}: tw4n holds
  // the first half circle, the second is its negation
  auto step_tw = [&](int r, int k1) -> double2 {
    const int q = (8 * r * k1) & (4 * N - 1);
    const double2 w = __ldg(&tw4n[q & (2 * N - 1)]);
    return q >= 2 * N ? make_double2(-w.x, -w.y) : w;
  };
  // the 16 output accumulators live in the thread's TMEM lane (32 columns;
  // 16 warps = 4 per lane quarter): no register spills around the FFT
  __shared__ uint32_t tmem_base;
  const int warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tF = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + 32u * (uint32_t)(warp >> 2);
  {
    uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) tm_st8(tF + 8 * q, z);
    tm_wait_st();
  }
  const int tp = CS * t + m1;  // Z index m = tp + (N/16) r: the pack's twiddle bases
  const double2 ta_t = __ldg(&tw4n[tp]);
  const double2 r4_t = __ldg(&tw4n[4 * tp]);
  cl.sync();  // every CTA's stage loaded (the first pack reads the mirror's)
  for (int m = 0; m < terms; ++m) {
    const bool odd = ((m & 1) ^ swap) != 0;
    double2 v[E];
#define FLB_CL_PACK(R)                                                                     \
  {                                                                                        \
    const int m2 = t + T * (R);                                                            \
    const int a_nm = m1 ? 2 * Q - 1 - m2 : (2 * Q - m2) & (2 * Q - 1);                     \
    const int a_pm = m1 ? Q - 1 - m2 : Q - m2;                                             \
    const double s_m = st[m2], s_mp = st[Q + m2], s_nm = rst[a_nm], s_pm = rst[a_pm];      \
    const bool m0 = m1 == 0 && m2 == 0;                                                    \
    v[R] = odd ? fwd_pack_vals<true, R>(s_m, s_mp, s_nm, s_pm, m0, ta_t, r4_t)             \
               : fwd_pack_vals<false, R>(s_m, s_mp, s_nm, s_pm, m0, ta_t, r4_t);           \
  }
    FLB_CL_PACK(0) FLB_CL_PACK(1) FLB_CL_PACK(2) FLB_CL_PACK(3)
    FLB_CL_PACK(4) FLB_CL_PACK(5) FLB_CL_PACK(6) FLB_CL_PACK(7)
#undef FLB_CL_PACK
    pass_compute<Q, E, 8, 1, true>(v, t, fftw);
    pass_store<Q, E, 8, 1>(v, Y, t);
    __syncthreads();
    mid_passes<Q, E, 8, Q, true, 0>(Y, t, fftw, 0);
    cl.sync();  // (1) every Y row final, every pack of this term done
    // the next stage T_{m+1}(x) c at the own entries (x = n/N)
#pragma unroll
    for (int i = 0; i < E; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = h * Q + t + T * i;
        const double x = (double)(CS * a + m1) / (double)N;
        const double cur = st[a];
        st[a] = m == 0 ? x * cur : fma(2.0 * x, cur, -pv[a]);
        pv[a] = cur;
      }
    // step C: the CS-point inverse DFTs across the cluster, then the unpack
    const double* w = wt + ((size_t)m * CS + m1) * 16 * T + t;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int k1 = m1 * KQ + t + d * T;
      double2 y[CS];
#pragma unroll
      for (int r = 0; r < CS; ++r) {
        const double2 a = cl.map_shared_rank(Y, r)[smem_pad(k1)];
        y[r] = r ? cmul(a, step_tw(r, k1)) : a;
      }
      dft_r<CS, true>(y);
      // this d's 2 CS outputs: slots 2 CS d .. (8 per TMEM x8 access of 4 doubles)
#pragma unroll
      for (int g = 0; g < CS / 2; ++g) {
        uint32_t fw[8];
        const uint32_t addr = tF + (uint32_t)(2 * (2 * CS * d + 4 * g));
        tm_ld8(addr, fw);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = 2 * CS * d + 4 * g + u, k2 = (4 * g + u) >> 1;
          const double val = (u & 1) ? y[k2].y : y[k2].x;
          split2(join2(&fw[2 * u]) + __ldg(w + (size_t)i * T) * val, &fw[2 * u]);
        }
        tm_st8(addr, fw);
      }
    }
    tm_wait_st();
    cl.sync();  // (2) every Y read and stage write done before the next term
  }
  double* dst = out + col * ld_out;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t fw[8];
    tm_ld8(tF + 8 * q, fw);
#pragma unroll
    for (int u = 0; u < 4; ++u) dst[cl_out_row<LOG2N>(m1, t, 4 * q + u)] = join2(&fw[2 * u]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem_base) : "memory");
}

// The cluster kernel's weights: wt[((m CS + s) 16 + i) T + t] = the term-m
// weight of output row cl_out_row(s, t, i), with the sine flavour's sign and
// the DST's (-1)^k output sign folded in.
template <int LOG2N>
__global__ void cluster_weight_table_kernel(const double* __restrict__ delta, int terms, int swap,
                                            double* __restrict__ wt) {
  using C = ClCfg<LOG2N>;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;  // (s 16 + i) T + t
  if (j >= C::N) return;
  const int t = j % C::T, si = j / C::T, i = si % 16, sct = si / 16;
  const int k = cl_out_row<LOG2N>(sct, t, i);
  const double y = (double)C::N * delta[k];
  for (int m = 0; m < terms; ++m) {
    const bool odd = ((m & 1) ^ swap) != 0;
    double w = ((swap && (m & 1)) ? -1.0 : 1.0) * bessel_weight(m, y);
    if (odd && (k & 1)) w = -w;
    wt[(size_t)m * C::N + j] = w;
  }
}

template <int LOG2N>
void launch_cluster_fwd(const double* in, size_t ld_in, double* out, size_t ld_out, size_t batch,
                        const FastNdct& p, int* nonfinite, cudaStream_t s) {
  using C = ClCfg<LOG2N>;
  auto kern = cluster_ndct_fwd_kernel<LOG2N>;
  FLB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  const double2* tw = tw4n_table(LOG2N);
  const double2* fftw = pass_twiddles(12);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(C::T);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  constexpr size_t kMaxCols = 65535 / C::CS;
  for (size_t c0 = 0; c0 < batch; c0 += kMaxCols) {
    const size_t nc = std::min(kMaxCols, batch - c0);
    cfg.gridDim = dim3((unsigned)(nc * C::CS));
    FLB_CUDA(cudaLaunchKernelEx(&cfg, kern, in + c0 * ld_in, ld_in, out + c0 * ld_out, ld_out,
                                p.bes_terms, p.swap, (const double*)p.cl_wf, tw, fftw, nonfinite));
    note_launch("cluster_ndct_fwd_kernel");
  }
}

template <int LOG2N>
__global__ void bessel_tables_kernel(const double* __restrict__ delta, int terms,
                                     double* __restrict__ wf, double* __restrict__ wt,
                                     double* __restrict__ tt, int swap) {
  using C = Cfg<LOG2N>;
  constexpr int N = C::N, T = C::T;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const double yf = (double)N * delta[fwd_own_row<LOG2N>(j % T, j / T)];
  const double yt = (double)N * delta[tr_entry<N>(j)];
  const double x = (double)tr_row<N>(j % T, j / T) / (double)N;
  double tm1 = 1.0, tm = x;  // T_{m-1}, T_m
  for (int m = 0; m < terms; ++m) {
    const double sg = (swap && (m & 1)) ? -1.0 : 1.0;  // sine flavour: odd terms change sign
    wf[(size_t)m * N + j] = sg * bessel_weight(m, yf);
    wt[(size_t)m * N + j] = sg * bessel_weight(m, yt);
    const double tv = m == 0 ? 1.0 : m == 1 ? x : tm;
    tt[(size_t)m * N + j] = tv;
    if (m >= 1) {  // advance to T_{m+1}
      const double nx = 2.0 * x * tm - tm1;
      tm1 = tm;
      tm = nx;
    }
  }
}

// ---------------------------------------------------------------------------
// N > 8192 (one column no longer fits a CTA): the same real-DCT packing per
// term, with the N/2-point FFT done by the multi-pass engine (fft_pow2,
// six-step through HBM / L2). Per term: pack kernel (reads c, applies
// (n/N)^l by repeated squaring), FFT, unpack kernel (applies
// sign_l (N delta_k)^l / l! and accumulates into f). Batched over columns.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ipow(double r, int l) {
  double acc = 1.0;
  while (l) {
    if (l & 1) acc *= r;
    r *= r;
    l >>= 1;
  }
  return acc;
}

// (N delta)^l / l!, the reference's running product order (ndct.hpp:108)
__device__ __forceinline__ double taylor_weight(double nd, int l) {
  double p = 1.0;
  for (int i = 1; i <= l; ++i) p *= nd / (double)i;
  return p;
}

// T_m(x) by the three-term recurrence (m small).
__device__ __forceinline__ double cheb_t(int m, double x) {
  if (m == 0) return 1.0;
  double a = 1.0, b = x;
  for (int i = 1; i < m; ++i) {
    const double c = 2.0 * x * b - a;
    a = b;
    b = c;
  }
  return b;
}

// Terms of one multi-pass NDCT call: plain (one DCT-III / DST-III pass,
// odd = plain_op), the Chebyshev expansion (cheb, with the sine flavour swap)
// or Taylor terms.
struct BigTerms {
  int plain, plain_op, cheb, swap;
};
__device__ __forceinline__ int big_odd(const BigTerms& bt, int l) {
  return bt.plain ? bt.plain_op : ((l & 1) ^ bt.swap);
}
// weight of output row k in term l, its sign folded in (bessel_weight /
// taylor_sign (N delta)^l / l!)
__device__ __forceinline__ double big_weight(const BigTerms& bt, int l, double y0) {
  if (bt.plain) return 1.0;
  if (bt.cheb) return ((bt.swap && (l & 1)) ? -1.0 : 1.0) * bessel_weight(l, y0);
  return (((l + 1) / 2) % 2 == 0 ? 1.0 : -1.0) * taylor_weight(y0, l);
}
// stage factor of entry j in term l: T_l(j/N) (Chebyshev) or (j/N)^l
__device__ __forceinline__ double big_row(const BigTerms& bt, int l, double x) {
  if (bt.plain) return 1.0;
  return bt.cheb ? cheb_t(l, x) : ipow(x, l);
}

// Per-call tables for terms [l0, l0 + nt): wt[t][k] = big_weight(l0 + t,
// N delta_k), rt[t][j] = big_row(l0 + t, j/N) (shared by all columns).
// 1 / i, i < 128: the Bessel series' divisions as products in the per-call
// tables (one series per term and entry: 2^26 entries x 7 terms took 4.8 ms
// per table launch with divisions)
__constant__ double kRecip[128];
bool recip_ready[64] = {};
void ensure_recip() {
  static std::mutex mu;
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && recip_ready[dev]) return;
  double h[128];
  h[0] = 0.0;
  for (int i = 1; i < 128; ++i) h[i] = 1.0 / (double)i;
  FLB_CUDA(cudaMemcpyToSymbol(kRecip, h, sizeof h));
  if (dev < 64) recip_ready[dev] = true;
}

// J_m(y) by its power series (|y| <= ~1 here), reciprocals from kRecip
__device__ __forceinline__ double bessel_j_tab(int m, double y) {
  const double h = 0.5 * y, h2 = h * h;
  double t = 1.0;
  for (int i = 1; i <= m; ++i) t *= h * kRecip[i];
  double sum = t;
  for (int k = 1; k < 40 && m + k < 128; ++k) {
    t *= -h2 * (kRecip[k] * kRecip[m + k]);
    sum += t;
    if (fabs(t) <= 1e-18 * fabs(sum)) break;
  }
  return sum;
}

__global__ void big_tables_kernel(size_t n, int l0, int nt, BigTerms bt,
                                  const double* __restrict__ delta, double* __restrict__ wt,
                                  double* __restrict__ rt) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double y0 = bt.plain ? 0.0 : (double)n * delta[j];
  const double x = (double)j / (double)n;
  // T_l(x) continued by its recurrence from l0 (the same operations as cheb_t)
  double ta = bt.cheb ? cheb_t(l0, x) : 0.0, tb = bt.cheb ? cheb_t(l0 + 1, x) : 0.0;
  for (int t = 0; t < nt; ++t) {
    const int l = l0 + t;
    double w;
    if (bt.plain) {
      w = 1.0;
    } else if (bt.cheb) {
      // bessel_weight with the tabulated series
      const double jv = bessel_j_tab(l, y0);
      w = (l & 1) == 0 ? (l == 0 ? 1.0 : 2.0) * (((l >> 1) & 1) ? -jv : jv)
                       : -2.0 * ((((l - 1) >> 1) & 1) ? -jv : jv);
      if (bt.swap && (l & 1)) w = -w;
    } else {
      w = big_weight(bt, l, y0);
    }
    wt[(size_t)t * n + j] = w;
    if (bt.cheb) {
      rt[(size_t)t * n + j] = ta;
      const double tc = 2.0 * x * tb - ta;
      ta = tb;
      tb = tc;
    } else {
      rt[(size_t)t * n + j] = big_row(bt, l, x);
    }
  }
}

// The forward weights in the order of the packed transforms' entries, for the
// unpack fused into the last FFT pass (fft.cuh: NdctUnpack): entry m of term
// t holds outputs kx (real part) and ky (imaginary part), wp[t][m] =
// (+-wt[t][kx], +-wt[t][ky]) with big_fwd_unpack_kernel's signs (odd terms
// negate the odd outputs).
__global__ void big_wp_kernel(size_t n, int l0, int nt, BigTerms bt, const double* __restrict__ wt,
                              double2* __restrict__ wp) {
  const size_t P = n / 2;
  const size_t m = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (m >= P) return;
  const size_t kx = m < P / 2 ? 4 * m : 2 * n - 4 * m - 1, ky = m < P / 2 ? 4 * m + 2 : 2 * n - 4 * m - 3;
  for (int t = 0; t < nt; ++t) {
    const double sg = (big_odd(bt, l0 + t) && (kx & 1)) ? -1.0 : 1.0;  // kx, ky share their parity
    wp[(size_t)t * P + m] = make_double2(sg * wt[(size_t)t * n + kx], sg * wt[(size_t)t * n + ky]);
  }
}

// Forward pack of all nt terms: Z[(t nc + col) P + m] from the stage
// rt[t][j] c_j (the real-DCT packing of the file header). One thread per m for
// every term: the four column entries and the three twiddles of m are read /
// evaluated once (per term they were half the kernel's time at C2).
// NC columns per thread: the twiddles and the stage factors rt[t][.] of m are
// shared by all columns.
template <int NC>
__global__ void big_fwd_pack_kernel(const double* __restrict__ in, size_t ld, size_t n, size_t nc,
                                    int l0, int nt, BigTerms bt, const double* __restrict__ rt,
                                    double2* __restrict__ Z, int* nonfinite) {
  const size_t P = n / 2;
  const size_t col = blockIdx.y * (size_t)NC;
  const double* c = in + col * ld;
  const double nd = (double)n;
  for (size_t m = blockIdx.x * (size_t)blockDim.x + threadIdx.x; m < P;
       m += (size_t)gridDim.x * blockDim.x) {
    // stage indices: m, n - m (none for m = 0), m + P, P - m
    double c0[NC], c1[NC], c2[NC], c3[NC];
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
      const double* cq = c + (size_t)cc * ld;
      c0[cc] = cq[m];
      c1[cc] = m ? cq[n - m] : 0.0;
      c2[cc] = cq[m + P];
      c3[cc] = cq[P - m];
      if (nonfinite && l0 == 0) {
        if (!isfinite(c0[cc]) || !isfinite(c2[cc])) atomicOr(nonfinite, 1);
      }
    }
    double sa, ca, sb, cb, s4, c4;
    sincospi((double)m / (2.0 * nd), &sa, &ca);        // e^{i pi m/(2N)}
    sincospi((double)(m + P) / (2.0 * nd), &sb, &cb);  // e^{i pi (m+P)/(2N)}
    sincospi(2.0 * (double)m / nd, &s4, &c4);          // e^{2 pi i m/N}
    for (int tz = 0; tz < nt; ++tz) {
      const int odd = big_odd(bt, l0 + tz);
      const double* rw = rt + (size_t)tz * n;
      const double r0 = rw[m], r1 = m ? rw[n - m] : 0.0, r2 = rw[m + P], r3 = rw[P - m];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const double st0 = c0[cc] * r0, st1 = m ? c1[cc] * r1 : 0.0, st2 = c2[cc] * r2,
                     st3 = c3[cc] * r3;
        // DCT-III: X(0) = st(0), X(j) = st(j)/2; DST-III: X(0) = 0, X(j) = st(N - j)/2
        const double xa = odd ? (m ? 0.5 * st1 : 0.0) : (m ? 0.5 * st0 : st0);
        const double xan = m ? 0.5 * (odd ? st0 : st1) : 0.0;
        const double xb = 0.5 * (odd ? st3 : st2), xbn = 0.5 * (odd ? st2 : st3);
        const double2 Wa = make_double2(ca * xa + sa * xan, sa * xa - ca * xan);
        const double2 Wb = make_double2(cb * xb + sb * xbn, sb * xb - cb * xbn);
        const double2 sm = make_double2(Wa.x + Wb.x, Wa.y + Wb.y);
        const double2 d = make_double2(Wa.x - Wb.x, Wa.y - Wb.y);
        const double2 dr = make_double2(d.x * c4 - d.y * s4, d.x * s4 + d.y * c4);
        Z[((size_t)tz * nc + col + cc) * P + m] = make_double2(sm.x - dr.y, sm.y + dr.x);
      }
    }
  }
}

// Forward unpack of all nt terms: f_k (+)= sum_t wt[t][k] y_t(k), one store.
__global__ void big_fwd_unpack_kernel(const double2* __restrict__ Z, size_t n, size_t nc, int l0,
                                      int nt, BigTerms bt, const double* __restrict__ wt,
                                      double* __restrict__ out, size_t ld, int first) {
  const size_t P = n / 2;
  const size_t col = blockIdx.y;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n;
       k += (size_t)gridDim.x * blockDim.x) {
    const size_t q = (k & 1) ? (n - 1 - (k >> 1)) : (k >> 1);
    double acc = 0.0;
    for (int t = 0; t < nt; ++t) {
      const double2 z = Z[((size_t)t * nc + col) * P + (q >> 1)];
      double y = (q & 1) ? z.y : z.x;
      if (big_odd(bt, l0 + t) && (k & 1)) y = -y;
      acc += wt[(size_t)t * n + k] * y;
    }
    double* o = out + col * ld + k;
    *o = first ? acc : *o + acc;
  }
}

// Transposed pack of term l0 + blockIdx.z: the weighted input h_k = wt[z][k]
// (mult_k) g_k (DST^T: odd entries negated), packed into Z.
__global__ void big_tr_pack_kernel(const double* __restrict__ in, size_t ld, size_t n, size_t nc,
                                   int l0, BigTerms bt, const double* __restrict__ wt,
                                   const double* __restrict__ mult, double2* __restrict__ Z,
                                   int* nonfinite) {
  const size_t P = n / 2;
  const size_t col = blockIdx.y;
  const int tz = blockIdx.z, l = l0 + tz;
  const int odd = big_odd(bt, l);
  const double* g = in + col * ld;
  const double* ww = wt + (size_t)tz * n;
  double2* Zc = Z + ((size_t)tz * nc + col) * P;
  auto h = [&](size_t k) -> double {
    double v = g[k];
    if (mult) v = mult[k] * v;
    v = ww[k] * v;
    return (odd && (k & 1)) ? -v : v;
  };
  auto V = [&](size_t q) -> double { return q < P ? h(2 * q) : h(2 * (n - 1 - q) + 1); };
  for (size_t m = blockIdx.x * (size_t)blockDim.x + threadIdx.x; m < P;
       m += (size_t)gridDim.x * blockDim.x) {
    if (nonfinite && l == 0) {
      double a = g[2 * m], b = g[2 * m + 1];
      if (mult) {
        a *= mult[2 * m];
        b *= mult[2 * m + 1];
      }
      if (!isfinite(a) || !isfinite(b)) atomicOr(nonfinite, 1);
    }
    Zc[m] = make_double2(V(2 * m), V(2 * m + 1));
  }
}

// The transposed pack fused into the first FFT pass (fft.cuh: NdctTrPack): the
// column's input (times mult) once in packed-entry order, G[col][m] =
// (v(kx), v(ky)); the per-term weights and signs are wp's (big_wp_kernel).
__global__ void big_tr_g_kernel(const double* __restrict__ in, size_t ld, size_t n,
                                const double* __restrict__ mult, double2* __restrict__ G,
                                int* nonfinite) {
  const size_t P = n / 2;
  const size_t col = blockIdx.y;
  const double* g = in + col * ld;
  for (size_t m = blockIdx.x * (size_t)blockDim.x + threadIdx.x; m < P;
       m += (size_t)gridDim.x * blockDim.x) {
    const size_t kx = m < P / 2 ? 4 * m : 2 * n - 4 * m - 1, ky = m < P / 2 ? 4 * m + 2 : 2 * n - 4 * m - 3;
    double a = g[kx], b = g[ky];
    if (mult) {
      a *= mult[kx];
      b *= mult[ky];
    }
    if (nonfinite && (!isfinite(a) || !isfinite(b))) atomicOr(nonfinite, 1);
    G[col * P + m] = make_double2(a, b);
  }
}

// Transposed unpack of all nt terms: out_r (+)= sum_t rt[t][r] X_t(r).
// The outputs r in {a, P - a, P + a, N - a} read the same two packed entries
// a, P - a of every term (DCT^T rows at kk = r, DST^T rows at kk = N - r): one
// thread per a in [0, P/2] computes all four with its twiddles evaluated once
// (per output and term they were half of the kernel's time at C2).
__device__ __forceinline__ double big_tr_value(double2 za, double2 zc, double c2, double s2, double ch,
                                               double sh) {
  const double2 ev = make_double2(0.5 * (za.x + zc.x), 0.5 * (za.y - zc.y));
  const double2 od = make_double2(0.5 * (za.y + zc.y), -0.5 * (za.x - zc.x));
  const double2 Vv = make_double2(ev.x + od.x * c2 - od.y * s2, ev.y + od.x * s2 + od.y * c2);
  return ch * Vv.x + sh * Vv.y;
}
// NC columns per thread (the twiddles and the row factors rt[t][r] are shared
// by all columns: per column they were as much L2 traffic as the packed rows).
template <int NC>
__global__ void big_tr_unpack_kernel(const double2* __restrict__ Z, size_t n, size_t nc, int l0,
                                     int nt, BigTerms bt, const double* __restrict__ rt,
                                     double* __restrict__ out, size_t ld, int first) {
  const size_t P = n / 2;
  const size_t col = blockIdx.y * (size_t)NC;
  const double nd = (double)n;
  for (size_t a = blockIdx.x * (size_t)blockDim.x + threadIdx.x; a <= P / 2;
       a += (size_t)gridDim.x * blockDim.x) {
    const size_t bq = (P - a) & (P - 1);
    const int nr = (a != 0 && a != P / 2) ? 4 : 2;
    const size_t r[4] = {a, P + a, P - a, 2 * P - a};
    double c2[4], s2[4], ch[4], sh[4], acc[NC][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) acc[cc][e] = 0.0;
      c2[e] = s2[e] = ch[e] = sh[e] = 0.0;
      if (e < nr) {
        sincospi(-2.0 * (double)r[e] / nd, &s2[e], &c2[e]);  // e^{-2 pi i r/N}
        sincospi((double)r[e] / (2.0 * nd), &sh[e], &ch[e]);  // e^{i pi r/(2N)}
      }
    }
    for (int t = 0; t < nt; ++t) {
      const int odd = big_odd(bt, l0 + t);
      const double2* Zc = Z + ((size_t)t * nc + col) * P;
      double2 za[NC], zb[NC];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        za[cc] = Zc[(size_t)cc * P + a];
        zb[cc] = Zc[(size_t)cc * P + bq];
      }
      const double* rw = rt + (size_t)t * n;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (e >= nr) break;
        // rows e >= 2 read the pair swapped; the DST^T rows use kk = N - r:
        // e^{-2 pi i kk/N} = conj, e^{i pi kk/(2N)} = i conj, and swap again
        const bool swp = (e >= 2) != (odd != 0);
        const double w = rw[r[e]];
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          const double2 p0 = swp ? zb[cc] : za[cc], p1 = swp ? za[cc] : zb[cc];
          double x;
          if (!odd)
            x = big_tr_value(p0, p1, c2[e], s2[e], ch[e], sh[e]);
          else
            x = r[e] == 0 ? 0.0 : big_tr_value(p0, p1, c2[e], -s2[e], sh[e], ch[e]);
          acc[cc][e] = __fma_rn(w, x, acc[cc][e]);
        }
      }
    }
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (e >= nr) break;
        double* o = out + (col + cc) * ld + r[e];
        *o = first ? acc[cc][e] : *o + acc[cc][e];
      }
  }
}

// N > 8192: every term's packed transform in one batched multi-pass FFT
// (terms x columns). The per-term weights / stage factors come from tables
// [terms][N] that a plan builds on its first call and keeps (per-call tables
// for the free functions). From N = 2^15: forward, the unpack runs inside the
// FFT's row pass (fft_pow2_ndct_unpack: all terms of a column per CTA, the
// weighted sum in registers, the transformed rows never written); transposed,
// the pack runs inside the first pass's loads (fft_pow2_ndct_tr_pack: the
// column's weighted input once in packed order times the packed-order
// weights). At N = 2^14 (one shared-memory FFT per row) the separate unpack /
// pack kernels run.
// Scratch of one batched multi-pass NDCT call (packed rows + FFT scratch):
// 8 GiB (2^26: 2 batches of 7 terms: NDCT 35.9 -> 32.0 ms, NDCT^T 42.4 ->
// 37.6 ms against 2 GiB; 16 GiB: 31.5 / 36.5 ms).
#ifndef FLB_BIG_BUDGET_GIB
#define FLB_BIG_BUDGET_GIB 8
#endif
constexpr size_t kBigBudget = size_t(FLB_BIG_BUDGET_GIB) << 30;
// largest pair of kept plan tables (2^26 x 14 terms: 15 GiB of the 180)
#ifndef FLB_BIG_TABLE_CACHE_GIB
#define FLB_BIG_TABLE_CACHE_GIB 16
#endif
constexpr size_t kBigTableCache = size_t(FLB_BIG_TABLE_CACHE_GIB) << 30;
#ifndef FLB_BIG_PACK_COLS
#define FLB_BIG_PACK_COLS 2  // columns per thread of the forward pack (C2 0.501 -> 0.478 ms; 4: 0.483)
#endif
#ifndef FLB_BIG_TR_COLS
#define FLB_BIG_TR_COLS 2  // columns per thread of the transposed unpack
#endif
#ifndef FLB_BIG_FUSED_UNPACK
#define FLB_BIG_FUSED_UNPACK 1
#endif

void launch_big(int log2n, int transpose, const double* in, size_t ld_in, double* out,
                size_t ld_out, size_t batch, const double* delta, int l_lo, int l_hi,
                int plain_op, const double* mult, int* nonfinite, cudaStream_t s, int cheb,
                int swap, const FastNdct* owner = nullptr) {
  const size_t n = size_t(1) << log2n, P = n / 2;
  if (ld_in != ld_out) fail(FL_RUNTIME_ERROR, "fast ndct: mismatched strides");
  const int plain = plain_op >= 0;
  if (plain) {
    l_lo = 0;
    l_hi = 1;
  }
  const BigTerms bt{plain, plain_op, cheb, swap};
  const int terms = l_hi - l_lo;
  if (terms <= 0) return;
  constexpr size_t kBudget = kBigBudget;  // Z + S bytes
  const size_t per_term_col = 2 * P * sizeof(double2);
  const size_t chunk = std::max<size_t>(1, std::min<size_t>(batch, kBudget / per_term_col));
  const int tb = (int)std::max<size_t>(1, std::min<size_t>(terms, kBudget / (per_term_col * chunk)));
  double2 *Z = nullptr, *S = nullptr;
  double *wt = nullptr, *rt = nullptr;
  FLB_CUDA(cudaMallocAsync(&Z, (size_t)tb * chunk * P * sizeof(double2), s));
  FLB_CUDA(cudaMallocAsync(&S, (size_t)tb * chunk * P * sizeof(double2), s));
  // a plan's tables of all its terms: built on the first call, then kept
  // (published after one synchronisation; other threads wait on the mutex)
  const double *wt_all = nullptr, *rt_all = nullptr;
  if (owner && cheb && !plain && !owner->async_alloc && delta == owner->delta &&
      owner->bes_terms > 0 && l_hi <= owner->bes_terms) {
    const size_t bytes = (size_t)owner->bes_terms * n * sizeof(double);
    std::lock_guard<std::mutex> lock(owner->big_mu);
    if (!owner->big_tried) {
      owner->big_tried = true;
      if (2 * bytes <= kBigTableCache) {
        double *w = nullptr, *r = nullptr;
        if (cudaMalloc(&w, bytes) == cudaSuccess && cudaMalloc(&r, bytes) == cudaSuccess) {
          ensure_recip();
          big_tables_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, 0, owner->bes_terms, bt,
                                                                        delta, w, r);
          note_launch("big_tables_kernel");
          FLB_CUDA(cudaStreamSynchronize(s));
          owner->big_wt = w;
          owner->big_rt = r;
        } else {
          if (w) cudaFree(w);
          cudaGetLastError();
        }
      }
    }
    wt_all = owner->big_wt;
    rt_all = owner->big_rt;
  }
  if (!wt_all) {
    FLB_CUDA(cudaMallocAsync(&wt, (size_t)tb * n * sizeof(double), s));
    FLB_CUDA(cudaMallocAsync(&rt, (size_t)tb * n * sizeof(double), s));
  }
  // forward: the unpack fused into the last FFT pass (packed-order weights)
  const bool fused_unpack = FLB_BIG_FUSED_UNPACK && fft_pow2_ndct_unpack_ok(log2n - 1) &&
                            (!transpose || (size_t)tb * chunk <= 65535);
  const double2* wp_all = nullptr;
  double2* wp = nullptr;
  if (fused_unpack && wt_all) {
    std::lock_guard<std::mutex> lock(owner->big_mu);
    if (!owner->big_wp_tried) {
      owner->big_wp_tried = true;
      double2* w = nullptr;
      if (cudaMalloc(&w, (size_t)owner->bes_terms * P * sizeof(double2)) == cudaSuccess) {
        big_wp_kernel<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(n, 0, owner->bes_terms, bt, wt_all, w);
        note_launch("big_wp_kernel");
        FLB_CUDA(cudaStreamSynchronize(s));
        owner->big_wp = w;
      } else {
        cudaGetLastError();
      }
    }
    wp_all = owner->big_wp;
  }
  if (fused_unpack && !wp_all) FLB_CUDA(cudaMallocAsync(&wp, (size_t)tb * P * sizeof(double2), s));
  double2* G = nullptr;  // transposed: the weighted input in packed order
  if (fused_unpack && transpose) FLB_CUDA(cudaMallocAsync(&G, chunk * P * sizeof(double2), s));
  const unsigned gx = (unsigned)std::min<size_t>((P + 255) / 256, 2048);
  const unsigned gxn = (unsigned)std::min<size_t>((n + 255) / 256, 4096);
  const unsigned gxq = (unsigned)std::min<size_t>((P / 2 + 256) / 256, 4096);
  for (int l0 = l_lo; l0 < l_hi; l0 += tb) {
    const int nt = std::min(tb, l_hi - l0);
    if (wt_all) {
      wt = const_cast<double*>(wt_all) + (size_t)l0 * n;
      rt = const_cast<double*>(rt_all) + (size_t)l0 * n;
      if (wp_all) wp = const_cast<double2*>(wp_all) + (size_t)l0 * P;
    } else {
      ensure_recip();
      big_tables_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, l0, nt, bt, delta, wt, rt);
      note_launch("big_tables_kernel");
    }
    if (fused_unpack && !wp_all) {
      big_wp_kernel<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(n, l0, nt, bt, wt, wp);
      note_launch("big_wp_kernel");
    }
    for (size_t c0 = 0; c0 < batch; c0 += chunk) {
      const size_t nc = batch - c0 < chunk ? batch - c0 : chunk;
      const int first = l0 == l_lo;
      if (!transpose) {
        if (nc % FLB_BIG_PACK_COLS == 0 && FLB_BIG_PACK_COLS > 1)
          big_fwd_pack_kernel<FLB_BIG_PACK_COLS><<<dim3(gx, (unsigned)(nc / FLB_BIG_PACK_COLS)), 256, 0, s>>>(
              in + c0 * ld_in, ld_in, n, nc, l0, nt, bt, rt, Z, nonfinite);
        else
          big_fwd_pack_kernel<1><<<dim3(gx, (unsigned)nc), 256, 0, s>>>(
              in + c0 * ld_in, ld_in, n, nc, l0, nt, bt, rt, Z, nonfinite);
        note_launch("big_fwd_pack_kernel");
        if (fused_unpack) {
          fft_pow2_ndct_unpack(Z, S, log2n - 1, true,
                               NdctUnpack{wp, out + c0 * ld_out, ld_out, nc, nt, first}, s);
        } else {
          fft_pow2(Z, S, log2n - 1, nc * nt, true, s);
          big_fwd_unpack_kernel<<<dim3(gxn, (unsigned)nc), 256, 0, s>>>(
              Z, n, nc, l0, nt, bt, wt, out + c0 * ld_out, ld_out, first);
          note_launch("big_fwd_unpack_kernel");
        }
      } else {
        if (fused_unpack) {
          // the pack fused into the first FFT pass's loads
          big_tr_g_kernel<<<dim3(gx, (unsigned)nc), 256, 0, s>>>(in + c0 * ld_in, ld_in, n, mult, G,
                                                                 l0 == l_lo ? nonfinite : nullptr);
          note_launch("big_tr_g_kernel");
          fft_pow2_ndct_tr_pack(Z, S, log2n - 1, false, NdctTrPack{wp, G, nc, nt}, s);
        } else {
          big_tr_pack_kernel<<<dim3(gx, (unsigned)nc, (unsigned)nt), 256, 0, s>>>(
              in + c0 * ld_in, ld_in, n, nc, l0, bt, wt, mult, Z, nonfinite);
          note_launch("big_tr_pack_kernel");
          fft_pow2(Z, S, log2n - 1, nc * nt, false, s);
        }
        if (nc % FLB_BIG_TR_COLS == 0 && FLB_BIG_TR_COLS > 1)
          big_tr_unpack_kernel<FLB_BIG_TR_COLS><<<dim3(gxq, (unsigned)(nc / FLB_BIG_TR_COLS)), 256, 0, s>>>(
              Z, n, nc, l0, nt, bt, rt, out + c0 * ld_out, ld_out, first);
        else
          big_tr_unpack_kernel<1><<<dim3(gxq, (unsigned)nc), 256, 0, s>>>(
              Z, n, nc, l0, nt, bt, rt, out + c0 * ld_out, ld_out, first);
        note_launch("big_tr_unpack_kernel");
      }
    }
  }
  cudaFreeAsync(Z, s);
  cudaFreeAsync(S, s);
  if (!wt_all) {
    cudaFreeAsync(wt, s);
    cudaFreeAsync(rt, s);
  }
  if (fused_unpack && !wp_all) cudaFreeAsync(wp, s);
  if (G) cudaFreeAsync(G, s);
}

void dispatch(int log2n, int transpose, const double* in, size_t ld_in, double* out,
              size_t ld_out, size_t batch, const double* delta, int num_terms, int plain_op,
              const double* mult, int* nonfinite, cudaStream_t s, int l_lo = 0, int l_hi = -1,
              const FastNdct* bes = nullptr) {
  const bool cheb = bes && bes->bes_terms > 0 && plain_op < 0;
  if (cheb) num_terms = bes->bes_terms;
  if (l_hi < 0) l_hi = num_terms;
#ifndef FLB_NDCT_CLUSTER
#define FLB_NDCT_CLUSTER 1
#endif
  // the cluster kernel wins where the multi-pass path has to cut the batch
  // into several scratch-sized pieces (all terms x columns beyond its
  // scratch): 16384 x 4096 8.8 vs 14.5 ms; elsewhere the multi-pass path (all
  // terms packed per thread, shared twiddles) ties or wins: 16384 x 256 0.66
  // vs 0.65, 32768 x 128 0.82 vs 0.68, 65536 x 128 1.98 vs 1.28, 65536 x 512
  // 7.6 vs 6.1 ms
  const size_t cs = (size_t(1) << log2n) / 8192;
  const bool cl_fill = batch * cs >= 2 * (size_t)sm_count() &&
                       (size_t)num_terms * batch * (size_t(16) << log2n) > kBigBudget;
  if (FLB_NDCT_CLUSTER && cheb && !transpose && bes->cl_wf && l_lo == 0 && l_hi == num_terms &&
      log2n >= 14 && log2n <= 15 && cl_fill) {
    if (log2n == 14)
      launch_cluster_fwd<14>(in, ld_in, out, ld_out, batch, *bes, nonfinite, s);
    else
      launch_cluster_fwd<15>(in, ld_in, out, ld_out, batch, *bes, nonfinite, s);
    return;
  }
  if (log2n > 13) {
    launch_big(log2n, transpose, in, ld_in, out, ld_out, batch, delta, l_lo, l_hi, plain_op, mult,
               nonfinite, s, cheb ? 1 : 0, cheb ? bes->swap : 0, bes);
    return;
  }
  if (plain_op < 0 && (l_lo != 0 || l_hi != num_terms))
    fail(FL_INVALID_ARGUMENT, "ndct: term subsets need N > 8192 (multi-pass path)");
  switch (log2n) {
    case 9: launch_fast<9>(transpose, in, ld_in, out, ld_out, batch, delta, num_terms, plain_op, mult, nonfinite, s, bes); break;
    case 10: launch_fast<10>(transpose, in, ld_in, out, ld_out, batch, delta, num_terms, plain_op, mult, nonfinite, s, bes); break;
    case 11: launch_fast<11>(transpose, in, ld_in, out, ld_out, batch, delta, num_terms, plain_op, mult, nonfinite, s, bes); break;
    case 12: launch_fast<12>(transpose, in, ld_in, out, ld_out, batch, delta, num_terms, plain_op, mult, nonfinite, s, bes); break;
    case 13: launch_fast<13>(transpose, in, ld_in, out, ld_out, batch, delta, num_terms, plain_op, mult, nonfinite, s, bes); break;
    default: fail(FL_RUNTIME_ERROR, "fast ndct: unsupported size");
  }
}

int log2_exact(size_t n) {
  if (n == 0 || (n & (n - 1))) return -1;
  int l = 0;
  while ((size_t(1) << l) < n) ++l;
  return l;
}

// Terms of the Chebyshev (Jacobi-Anger) expansion with the same perturbation
// bound as cheb1_terms (|N delta| <= 0.83845): smallest M with
// 2 sum_{m >= M} |J_m(0.83845)| <= tol (|T_m| <= 1 on [0, 1]); 14 at 2^-52
// against Taylor's 17.
int bessel_terms_at(double y, double tol) {
  if (!(tol > 0.0 && tol < 1.0) || !(y >= 0.0 && y <= 2.0)) return -1;
  for (int M = 1; M <= 30; ++M) {
    double tail = 0.0;
    for (int m = M; m < M + 12; ++m) tail += 2.0 * fabs(bessel_j(m, y));
    if (tail <= tol) return M;
  }
  return -1;
}

int bessel_terms(double tol) { return bessel_terms_at(0.83845, tol); }

int cheb1_terms(double tol) {  // ndct.hpp:49-59 for cheb1; -1 if unattainable
  if (!(tol > 0.0 && tol < 1.0)) return -1;
  double b = 1.0;
  for (int l = 1; l <= 30; ++l) {
    b *= 0.83845 / (double)l;
    if (b <= tol) return l;
  }
  return -1;
}

}  // namespace

bool fast_trig_ok(size_t n, int kind) {
  const int lg = log2_exact(n);
  return kind == FL_CHEB1 && lg >= kFastMinLog2 && lg <= kFastMaxLog2;
}

void fast_trig(int op, size_t n, const double* in, double* out, size_t batch, size_t ld,
               cudaStream_t s) {
  const int transpose = op == FL_DCT_III_T || op == FL_DST_III_T;
  const int plain = (op == FL_DST_III || op == FL_DST_III_T) ? 1 : 0;
  dispatch(log2_exact(n), transpose, in, ld, out, ld, batch, nullptr, 1, plain, nullptr, nullptr, s);
}

bool fast_ndct_literal_ok(size_t n, int kind) { return fast_trig_ok(n, kind); }

bool fast_trig_bessel_ok(size_t n, int kind) {
  const int lg = log2_exact(n);
  return kind == FL_CHEBSTAR && lg >= kFastMinLog2 && lg <= kFastMaxLog2;
}

// dct_iii / dst_iii / *_transpose on the chebstar grid (trig.hpp:55-136) at
// power-of-two N: the chebstar angles are cheb1 angles plus an exact offset
// (|N offset| < pi/4), so the length-(2N+1) transform becomes the fused
// Chebyshev-expansion NDCT about cheb1 with zero node offsets (the sine
// flavour for the DSTs).
void fast_trig_bessel(int op, size_t n, const double* in, double* out, size_t batch, size_t ld,
                      cudaStream_t s) {
  const int transpose = op == FL_DCT_III_T || op == FL_DST_III_T;
  const int swap = (op == FL_DST_III || op == FL_DST_III_T) ? 1 : 0;
  FastNdctHolder h;
  h.p = fast_ndct_create_bessel(n, FL_CHEBSTAR, nullptr, 1, swap, s);
  if (!h.p) fail(FL_RUNTIME_ERROR, "fast trig: chebstar expansion unavailable");
  fast_ndct_run(*h.p, transpose, in, ld, out, ld, batch, nullptr, nullptr, s);
}

FastNdct* fast_ndct_create_literal(size_t n, int kind, int num_terms, const double* delta,
                                   cudaStream_t) {
  if (!fast_ndct_literal_ok(n, kind)) return nullptr;
  FastNdct* p = new FastNdct;
  p->n = n;
  p->log2n = log2_exact(n);
  p->num_terms = num_terms;
  p->delta = delta;
  return p;
}

// delta'_k = delta_k + (theta*_kind(k) - theta0_k): the angle the reference
// evaluates for kind (its exact grid angle plus the fp64 offset delta_k,
// ndct.hpp:98-117) re-expressed about the cheb1 angle theta0_k = (k + 1/2) pi / N.
// The grid offset is exact up to one rounding: (k + 3/4) pi / (N + 1/2) -
// (k + 1/2) pi / N = (N - 2k - 1) pi / (2N (2N + 1)). (Subtracting the two
// rounded angles instead would move the evaluation point by their rounding
// errors, ~1e-16 rad, i.e. ~N 1e-16 relative at degree N.) delta may be null
// (zero offsets: the plain chebstar DCT). amax[0] = max |delta|, amax[1] =
// max |delta'| (bit patterns of non-negative doubles order as integers).
__global__ void fast_delta_kernel(size_t n, int kind, const double* __restrict__ delta,
                                  double* __restrict__ out, unsigned long long* amax) {
  const size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  double d = 0.0, dp = 0.0;
  if (k < n) {
    d = delta ? delta[k] : 0.0;
    double off = 0.0;
    if (kind == FL_CHEBSTAR) {
      const double nd = (double)n;
      off = (double)((long long)n - 2 * (long long)k - 1) * (kPi / (2.0 * nd * (2.0 * nd + 1.0)));
    }
    dp = d + off;
    out[k] = dp;
  }
  if (amax) {
    // one atomic pair per warp (one per thread serialised on the two
    // addresses: 91 us at N = 65536); a NaN offset has the largest bit pattern
    unsigned long long a = (unsigned long long)__double_as_longlong(fabs(d));
    unsigned long long b = (unsigned long long)__double_as_longlong(fabs(dp));
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long a2 = __shfl_xor_sync(0xffffffffu, a, o);
      const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, b, o);
      a = a2 > a ? a2 : a;
      b = b2 > b ? b2 : b;
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&amax[0], a);
      atomicMax(&amax[1], b);
    }
  }
}

void build_bessel_tables(FastNdct* p, int M, cudaStream_t s) {
  const size_t n = p->n;
  for (double** t : {&p->bes_wf, &p->bes_wt, &p->bes_tt}) {
    if (p->async_alloc)
      FLB_CUDA(cudaMallocAsync(t, (size_t)M * n * sizeof(double), s));
    else
      FLB_CUDA(cudaMalloc(t, (size_t)M * n * sizeof(double)));
  }
  const unsigned grid = (unsigned)((n + 255) / 256);
  switch (p->log2n) {
#define FLB_BES(LG)                                                                        \
  case LG:                                                                                 \
    bessel_tables_kernel<LG><<<grid, 256, 0, s>>>(p->delta, M, p->bes_wf, p->bes_wt,       \
                                                  p->bes_tt, p->swap);                     \
    break;
    FLB_BES(9) FLB_BES(10) FLB_BES(11) FLB_BES(12) FLB_BES(13)
#undef FLB_BES
  }
  note_launch("bessel_tables_kernel");
}

// The cluster kernel's weight table (N = 2^14, 2^15, forward: the sizes the
// dispatch may pick it for).
void build_cluster_table(FastNdct* p, int M, cudaStream_t s) {
  if (p->log2n < 14 || p->log2n > 15) return;
  const size_t n = p->n;
  if (p->async_alloc)
    FLB_CUDA(cudaMallocAsync(&p->cl_wf, (size_t)M * n * sizeof(double), s));
  else
    FLB_CUDA(cudaMalloc(&p->cl_wf, (size_t)M * n * sizeof(double)));
  const unsigned grid = (unsigned)((n + 255) / 256);
  switch (p->log2n) {
    case 14: cluster_weight_table_kernel<14><<<grid, 256, 0, s>>>(p->delta, M, p->swap, p->cl_wf); break;
    default: cluster_weight_table_kernel<15><<<grid, 256, 0, s>>>(p->delta, M, p->swap, p->cl_wf); break;
  }
  note_launch("cluster_weight_table_kernel");
}

FastNdct* fast_ndct_create(size_t n, double tol, int kind, const double* delta) {
  const int lg = log2_exact(n);
  if (lg < kFastMinLog2 || lg > kFastMaxLog2) return nullptr;
  const int L = cheb1_terms(tol);
  if (L < 0) return nullptr;
  FastNdct* p = new FastNdct;
  p->n = n;
  p->log2n = lg;
  p->num_terms = L;
  FLB_CUDA(cudaMalloc(&p->owned_delta, n * sizeof(double)));
  fast_delta_kernel<<<(unsigned)((n + 255) / 256), 256>>>(n, kind, delta, p->owned_delta, nullptr);
  note_launch("fast_delta_kernel");
  p->delta = p->owned_delta;
#ifndef FLB_NDCT_BESSEL
#define FLB_NDCT_BESSEL 1
#endif
  // |N delta'| <= pi/4 + 1/(6 pi) = 0.83845 for Legendre nodes on either grid
  // (the cheb1 bound of ndct.hpp:38-44): the term count of that bound
  const int M = bessel_terms(tol);
  if (FLB_NDCT_BESSEL && M > 0 && M < L) p->bes_terms = M;  // multi-pass: weights on the fly
  if (FLB_NDCT_BESSEL && lg <= 13 && M > 0 && M < L) build_bessel_tables(p, M, 0);
  if (p->bes_terms > 0) build_cluster_table(p, M, 0);
  return p;
}

FastNdct* fast_ndct_create_bessel(size_t n, int kind, const double* delta, int num_terms,
                                  int swap, cudaStream_t s) {
  const int lg = log2_exact(n);
  if (lg < kFastMinLog2 || lg > kFastMaxLog2 || num_terms <= 0) return nullptr;
  FastNdct* p = new FastNdct;
  p->n = n;
  p->log2n = lg;
  p->swap = swap;
  p->alloc_stream = s;
  p->async_alloc = true;
  unsigned long long* amax = nullptr;
  FLB_CUDA(cudaMallocAsync(&p->owned_delta, n * sizeof(double), s));
  FLB_CUDA(cudaMallocAsync(&amax, 2 * sizeof(unsigned long long), s));
  FLB_CUDA(cudaMemsetAsync(amax, 0, 2 * sizeof(unsigned long long), s));
  fast_delta_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, kind, delta, p->owned_delta,
                                                                amax);
  note_launch("fast_delta_kernel");
  p->delta = p->owned_delta;
  unsigned long long h[2];
  FLB_CUDA(cudaMemcpyAsync(h, amax, sizeof h, cudaMemcpyDeviceToHost, s));
  FLB_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(amax, s);
  double dmax, ymax;
  memcpy(&dmax, &h[0], 8);
  memcpy(&ymax, &h[1], 8);
  // eligible when the literal evaluation is exact to fp64 rounding: its
  // truncation bound min((N max|delta|)^L / L!, C(L)) (ndct.hpp:147-155) at
  // or below 2^-52, and delta not identically zero (delta = 0 keeps the
  // literal path, bit-identical to dct_iii, test_ndct.cpp:112-125)
  const double nd = (double)n, q = nd * dmax;
  double node_bound = 1.0, grid_bound = 1.0;
  const double qq = kind == FL_CHEB1 ? 0.83845 : 1.0 / (6.0 * kPi);
  for (int l = 1; l <= num_terms; ++l) {
    node_bound *= q / (double)l;
    grid_bound *= qq / (double)l;
  }
  const double eps52 = 2.220446049250313e-16;
  const int M = bessel_terms_at(nd * ymax, eps52);
  const bool literal_exact = std::min(node_bound, grid_bound) <= eps52;
  const bool zero = delta != nullptr && dmax == 0.0;
  if (!(literal_exact && !zero && M > 0 && std::isfinite(ymax))) {
    fast_ndct_destroy(p);
    return nullptr;
  }
  p->num_terms = M;
  p->bes_terms = M;
  if (lg <= 13) build_bessel_tables(p, M, s);
  build_cluster_table(p, M, s);
  return p;
}

void fast_ndct_destroy(FastNdct* p) {
  if (!p) return;
  if (p->big_wt) cudaFree(p->big_wt);
  if (p->big_rt) cudaFree(p->big_rt);
  if (p->big_wp) cudaFree(p->big_wp);
  for (double* t : {p->owned_delta, p->bes_wf, p->bes_wt, p->bes_tt, p->cl_wf}) {
    if (!t) continue;
    if (p->async_alloc)
      cudaFreeAsync(t, p->alloc_stream);
    else
      cudaFree(t);
  }
  delete p;
}

void fast_ndct_run(const FastNdct& p, int transpose, const double* in, size_t ld_in, double* out,
                   size_t ld_out, size_t batch, const double* in_mult, int* nonfinite,
                   cudaStream_t s, int l_lo, int l_hi) {
  dispatch(p.log2n, transpose, in, ld_in, out, ld_out, batch, p.delta, p.num_terms, -1, in_mult,
           nonfinite, s, l_lo, l_hi, &p);
}

}  // namespace flb

namespace flb {
int fast_ndct_terms(const FastNdct& p) { return p.bes_terms > 0 ? p.bes_terms : p.num_terms; }
int fast_ndct_dlt_terms(const FastNdct& p) { return fast_ndct_terms(p); }
}  // namespace flb

// ===========================================================================
// Distributed four-step NDCT (dist_ndct.cuh): the multi-pass path's pack /
// unpack arithmetic (big_*_kernel) over the rank-local layouts of a four-step
// N/2-point FFT whose two FFT stages are separated by one all-to-all.
// ===========================================================================
#include "dist_ndct.cuh"

namespace flb {

struct FsLayout {
  size_t n = 0, L = 0, L1 = 0, L2 = 0, KB = 0, B = 0, U = 0;
  int log2n = 0, log2L1 = 0, log2L2 = 0, log2KB = 0;
  int world = 1, rank = 0, device = 0;
  std::vector<int> nres, cum;  // residues per rank, prefix sums (world + 1)
  size_t res_max = 0;
  int* d_res_all = nullptr;  // [world][res_max], -1 padded
  int* d_mirror = nullptr;   // [nres_me]: local index of (L1 - res) mod L1
  int* d_owner = nullptr;    // [L1]: rank owning residue m1
  int* d_lidx = nullptr;     // [L1]: its index in the owner's list
  int* d_cum = nullptr;      // [world + 1]
  int* d_nres = nullptr;     // [world]
  // per-rank weight table of the value side, wt[l][k1][k2l][b] = the
  // Chebyshev-expansion weight of term l at output k(p, b) (built on first
  // use for one FastNdct: terms x N/P doubles)
  mutable double* wt = nullptr;
  mutable const FastNdct* wt_for = nullptr;
  mutable std::mutex wt_mu;
  const int* res_me() const { return d_res_all + (size_t)rank * res_max; }
};

namespace {

constexpr int kFsTile = 32, kFsRows = 8;

struct FsDev {  // by-value kernel view of a layout
  unsigned long long n, L, L1, L2, KB, B, U;
  int log2L1, log2L2, log2KB, world, rank, nres_me;
  unsigned long long res_max;
  const int *res_all, *mirror, *owner, *lidx, *cum, *nres;
};
FsDev fs_dev(const FsLayout& f) {
  return FsDev{f.n, f.L, f.L1, f.L2, f.KB, f.B, f.U, f.log2L1, f.log2L2, f.log2KB, f.world, f.rank,
               f.nres[f.rank], f.res_max, f.d_res_all, f.d_mirror, f.d_owner, f.d_lidx, f.d_cum,
               f.d_nres};
}

// value side: output index k of packed slot q (the forward unpack's map)
__device__ __forceinline__ unsigned long long fs_k_of_q(const FsDev& d, unsigned long long q) {
  return q < d.L ? 2 * q : 2 * (d.n - 1 - q) + 1;
}
// first p (= k2 + L2 k1) of block `blk`'s even (g = 0) / odd (g = 1) range
__device__ __forceinline__ unsigned long long fs_p0(const FsDev& d, unsigned long long blk, int g) {
  return g ? d.L - (blk + 1) * (d.B / 4) : blk * (d.B / 4);
}
// position of slot pair (p, b = 0) in the value exchange layout of the pair
// (block owner dst, k2-block owner src): [src or dst][g][u][k2l][b]
__device__ __forceinline__ unsigned long long fs_xpos(const FsDev& d, unsigned long long peer,
                                                      unsigned long long blk, int g,
                                                      unsigned long long k1,
                                                      unsigned long long k2l) {
  const unsigned long long u = k1 - fs_p0(d, blk, g) / d.L2;
  return peer * (d.B / d.world) + (((unsigned long long)g * d.U + u) * d.KB + k2l) * 2;
}

// the Chebyshev-expansion weight of term l at y0 = N delta_k (big_tables_kernel)
__device__ __forceinline__ double fs_weight(int l, double y0, int swap) {
  const double jv = bessel_j_tab(l, y0);
  double w = (l & 1) == 0 ? (l == 0 ? 1.0 : 2.0) * (((l >> 1) & 1) ? -jv : jv)
                          : -2.0 * ((((l - 1) >> 1) & 1) ? -jv : jv);
  if (swap && (l & 1)) w = -w;
  return w;
}

// natural full vector <-> [dest][res_max][2 L2] (tile transpose: residues x j)
template <bool TO>
__global__ void fs_residue_kernel(FsDev d, const double* __restrict__ src, double* __restrict__ dst) {
  __shared__ double tile[kFsTile][kFsTile + 1];
  const unsigned long long J = 2 * d.L2;
  const int dest = blockIdx.z;
  const unsigned long long i0 = (unsigned long long)blockIdx.y * kFsTile;
  const unsigned long long j0 = (unsigned long long)blockIdx.x * kFsTile;
  const int* res = d.res_all + (size_t)dest * d.res_max;
  const unsigned long long base = (unsigned long long)dest * d.res_max * J;
  if (TO) {
    // read along residues (threads over i), write along j
    for (int jj = threadIdx.y; jj < kFsTile; jj += kFsRows) {
      const unsigned long long i = i0 + threadIdx.x, j = j0 + jj;
      double v = 0.0;
      if (i < d.res_max && j < J) {
        const int r = res[i];
        if (r >= 0) v = src[(unsigned long long)r + d.L1 * j];
      }
      tile[jj][threadIdx.x] = v;
    }
    __syncthreads();
    for (int ii = threadIdx.y; ii < kFsTile; ii += kFsRows) {
      const unsigned long long i = i0 + ii, j = j0 + threadIdx.x;
      if (i < d.res_max && j < J) dst[base + i * J + j] = tile[threadIdx.x][ii];
    }
  } else {
    for (int ii = threadIdx.y; ii < kFsTile; ii += kFsRows) {
      const unsigned long long i = i0 + ii, j = j0 + threadIdx.x;
      tile[ii][threadIdx.x] = (i < d.res_max && j < J) ? src[base + i * J + j] : 0.0;
    }
    __syncthreads();
    for (int jj = threadIdx.y; jj < kFsTile; jj += kFsRows) {
      const unsigned long long i = i0 + threadIdx.x, j = j0 + jj;
      if (i < d.res_max && j < J) {
        const int r = res[i];
        if (r >= 0) dst[(unsigned long long)r + d.L1 * j] = tile[threadIdx.x][jj];
      }
    }
  }
}

// forward pack of terms [t0, t0 + nt) for this rank's residues: Z[t][i][m2]
// for m = res_i + L1 m2 (big_fwd_pack_kernel's arithmetic)
__global__ void fs_fwd_pack_kernel(FsDev d, const double* __restrict__ chat, int t0, int nt,
                                   BigTerms bt, double2* __restrict__ Z, int* nonfinite) {
  const unsigned long long J = 2 * d.L2;
  const unsigned long long total = (unsigned long long)d.nres_me * d.L2;
  const int* res_me = d.res_all + (size_t)d.rank * d.res_max;
  const double nd = (double)d.n;
  for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
       e += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long i = e >> d.log2L2, m2 = e & (d.L2 - 1);
    const unsigned long long res = (unsigned long long)res_me[i];
    const unsigned long long m = res + d.L1 * m2;
    const double* ci = chat + i * J;
    const double c0 = ci[m2], c2 = ci[m2 + d.L2];
    double c1, c3;
    if (res == 0) {
      c1 = m2 ? ci[J - m2] : 0.0;
      c3 = ci[d.L2 - m2];
    } else {
      const double* cm = chat + (unsigned long long)d.mirror[i] * J;
      c1 = cm[J - 1 - m2];
      c3 = cm[d.L2 - 1 - m2];
    }
    if (nonfinite && t0 == 0) {
      if (!isfinite(c0) || !isfinite(c2)) atomicOr(nonfinite, 1);
    }
    const unsigned long long P = d.L;
    double sa, ca, sb, cb, s4, c4;
    sincospi((double)m / (2.0 * nd), &sa, &ca);
    sincospi((double)(m + P) / (2.0 * nd), &sb, &cb);
    sincospi(2.0 * (double)m / nd, &s4, &c4);
    // T_l of the four stage indices by the recurrence (cheb_t's operations)
    const double x0 = (double)m / nd, x1 = (double)(d.n - m) / nd, x2 = (double)(m + P) / nd,
                 x3 = (double)(P - m) / nd;
    double a0 = 1.0, a1 = 1.0, a2 = 1.0, a3 = 1.0;  // T_{l-1}
    double b0 = x0, b1 = x1, b2 = x2, b3 = x3;      // T_l
    double r0 = 1.0, r1 = 1.0, r2 = 1.0, r3 = 1.0;  // T at the current term
    for (int l = 0; l < t0 + nt; ++l) {
      if (bt.cheb) {
        if (l == 0) {
          r0 = r1 = r2 = r3 = 1.0;
        } else if (l == 1) {
          r0 = x0; r1 = x1; r2 = x2; r3 = x3;
        } else {
          const double n0 = 2.0 * x0 * b0 - a0, n1 = 2.0 * x1 * b1 - a1, n2 = 2.0 * x2 * b2 - a2,
                       n3 = 2.0 * x3 * b3 - a3;
          a0 = b0; a1 = b1; a2 = b2; a3 = b3;
          b0 = n0; b1 = n1; b2 = n2; b3 = n3;
          r0 = b0; r1 = b1; r2 = b2; r3 = b3;
        }
      } else {
        r0 = big_row(bt, l, x0); r1 = big_row(bt, l, x1); r2 = big_row(bt, l, x2); r3 = big_row(bt, l, x3);
      }
      if (l < t0) continue;
      const int tz = l - t0;
      const int odd = big_odd(bt, l);
      const double st0 = c0 * r0, st1 = m ? c1 * r1 : 0.0, st2 = c2 * r2, st3 = c3 * r3;
      const double xa = odd ? (m ? 0.5 * st1 : 0.0) : (m ? 0.5 * st0 : st0);
      const double xan = m ? 0.5 * (odd ? st0 : st1) : 0.0;
      const double xb = 0.5 * (odd ? st3 : st2), xbn = 0.5 * (odd ? st2 : st3);
      const double2 Wa = make_double2(ca * xa + sa * xan, sa * xa - ca * xan);
      const double2 Wb = make_double2(cb * xb + sb * xbn, sb * xb - cb * xbn);
      const double2 sm = make_double2(Wa.x + Wb.x, Wa.y + Wb.y);
      const double2 df = make_double2(Wa.x - Wb.x, Wa.y - Wb.y);
      const double2 dr = make_double2(df.x * c4 - df.y * s4, df.x * s4 + df.y * c4);
      Z[((unsigned long long)tz * d.nres_me + i) * d.L2 + m2] = make_double2(sm.x - dr.y, sm.y + dr.x);
    }
  }
}

// rows [t][i][k2] (after the L2-point inverse FFTs) times e^{+2 pi i res_i k2/L},
// into the exchange buffer [dest][t][i][k2l] (dest = k2 / KB)
__global__ void fs_fwd_twiddle_kernel(FsDev d, const double2* __restrict__ Z, int nt,
                                      double2* __restrict__ send) {
  const unsigned long long total = (unsigned long long)nt * d.nres_me * d.L2;
  const int* res_me = d.res_all + (size_t)d.rank * d.res_max;
  const unsigned long long chunk = (unsigned long long)nt * d.nres_me * d.KB;
  for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
       e += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long row = e >> d.log2L2, k2 = e & (d.L2 - 1);
    const unsigned long long i = row % (unsigned long long)d.nres_me;
    const unsigned long long ph = (unsigned long long)res_me[i] * k2;  // < L
    double s, c;
    sincospi(2.0 * (double)ph / (double)d.L, &s, &c);
    const double2 v = cmul(Z[e], make_double2(c, s));
    send[(k2 >> d.log2KB) * chunk + row * d.KB + (k2 & (d.KB - 1))] = v;
  }
}

// exchange buffer (from every source s: [t][i_s][k2l]) -> rows [t][k2l][m1]
__global__ void fs_fwd_gather_kernel(FsDev d, const double2* __restrict__ recv, int nt,
                                     double2* __restrict__ rows) {
  __shared__ double2 tile[kFsTile][kFsTile + 1];
  const int t = blockIdx.z;
  const unsigned long long m10 = (unsigned long long)blockIdx.x * kFsTile;
  const unsigned long long k0 = (unsigned long long)blockIdx.y * kFsTile;
  for (int mm = threadIdx.y; mm < kFsTile; mm += kFsRows) {
    const unsigned long long m1 = m10 + mm, k2l = k0 + threadIdx.x;
    double2 v = make_double2(0.0, 0.0);
    if (m1 < d.L1 && k2l < d.KB) {
      const int s = d.owner[m1];
      v = recv[(unsigned long long)d.cum[s] * d.KB * nt +
               ((unsigned long long)t * d.nres[s] + d.lidx[m1]) * d.KB + k2l];
    }
    tile[mm][threadIdx.x] = v;
  }
  __syncthreads();
  for (int kk = threadIdx.y; kk < kFsTile; kk += kFsRows) {
    const unsigned long long m1 = m10 + threadIdx.x, k2l = k0 + kk;
    if (m1 < d.L1 && k2l < d.KB)
      rows[((unsigned long long)t * d.KB + k2l) * d.L1 + m1] = tile[threadIdx.x][kk];
  }
}

// rows [t][k2l][k1] (after the L1-point inverse FFTs) -> the weighted sum over
// the group's terms at the two outputs of each slot pair, into the value
// exchange layout [dest block][g][u][k2l][b]
__global__ void fs_fwd_unpack_kernel(FsDev d, const double2* __restrict__ rows, int t0, int nt,
                                     BigTerms bt, const double2* __restrict__ wt,
                                     double* __restrict__ fx, int first) {
  __shared__ double2 tile[kFsTile][kFsTile + 1];
  constexpr int IT = kFsTile / kFsRows;
  const unsigned long long k10 = (unsigned long long)blockIdx.x * kFsTile;
  const unsigned long long k20 = (unsigned long long)blockIdx.y * kFsTile;
  // this thread's items: k2l = k20 + threadIdx.x, k1 = k10 + threadIdx.y + 8 it
  const unsigned long long k2l = k20 + threadIdx.x;
  unsigned long long k0[IT];
  double acc[IT][2];
  bool ok[IT];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const unsigned long long k1 = k10 + threadIdx.y + kFsRows * it;
    ok[it] = k1 < d.L1 && k2l < d.KB;
    const unsigned long long p = (unsigned long long)d.rank * d.KB + k2l + d.L2 * k1;
    k0[it] = ok[it] ? fs_k_of_q(d, 2 * p) : 0;  // both outputs of the pair have k's parity
    acc[it][0] = acc[it][1] = 0.0;
  }
  for (int t = 0; t < nt; ++t) {
    __syncthreads();
    for (int ii = threadIdx.y; ii < kFsTile; ii += kFsRows) {  // read along k1
      const unsigned long long r = k20 + ii, k1 = k10 + threadIdx.x;
      tile[ii][threadIdx.x] = (r < d.KB && k1 < d.L1)
                                  ? rows[((unsigned long long)t * d.KB + r) * d.L1 + k1]
                                  : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int l = t0 + t;
    const int odd = big_odd(bt, l);
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      if (!ok[it]) continue;
      const unsigned long long k1 = k10 + threadIdx.y + kFsRows * it;
      const double2 z = tile[threadIdx.x][threadIdx.y + kFsRows * it];
      const double2 w = wt[((unsigned long long)l * d.L1 + k1) * d.KB + k2l];
      const double sg = (odd && (k0[it] & 1)) ? -1.0 : 1.0;
      acc[it][0] += w.x * (sg * z.x);
      acc[it][1] += w.y * (sg * z.y);
    }
  }
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    if (!ok[it]) continue;
    const unsigned long long k1 = k10 + threadIdx.y + kFsRows * it;
    const unsigned long long k = k0[it];
    const unsigned long long blk = k / d.B;
    const int g = (int)(k & 1);
    double2* o = reinterpret_cast<double2*>(fx + fs_xpos(d, blk, blk, g, k1, k2l));
    const double2 v = make_double2(acc[it][0], acc[it][1]);
    if (first) {
      *o = v;
    } else {
      const double2 old = *o;
      *o = make_double2(old.x + v.x, old.y + v.y);
    }
  }
}

// the value side's weight table (see FsLayout::wt): per slot pair all terms
// (big_tables_kernel's series)
__global__ void fs_weights_kernel(FsDev d, const double* __restrict__ delta, int terms, BigTerms bt,
                                  double2* __restrict__ wt) {
  const unsigned long long total = d.L1 * d.KB;
  for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
       e += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long k1 = e >> d.log2KB, k2l = e & (d.KB - 1);
    const unsigned long long p = (unsigned long long)d.rank * d.KB + k2l + d.L2 * k1;
    const double ya = (double)d.n * delta[fs_k_of_q(d, 2 * p)];
    const double yb = (double)d.n * delta[fs_k_of_q(d, 2 * p + 1)];
    for (int l = 0; l < terms; ++l) {
      const double wa = bt.plain ? 1.0 : bt.cheb ? fs_weight(l, ya, bt.swap) : big_weight(bt, l, ya);
      const double wb = bt.plain ? 1.0 : bt.cheb ? fs_weight(l, yb, bt.swap) : big_weight(bt, l, yb);
      wt[(unsigned long long)l * total + e] = make_double2(wa, wb);
    }
  }
}

// value exchange layout <-> this rank's natural block (rank = the block owner;
// chunk s holds the slots of source / destination s's k2 block)
template <bool TO_BLOCK>
__global__ void fs_values_kernel(FsDev d, const double* __restrict__ src, double* __restrict__ dst) {
  const unsigned long long per = d.B / d.world;
  for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < d.B;
       e += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long s = e / per, rem = e - s * per;
    const int b = (int)(rem & 1);
    const unsigned long long r2 = rem >> 1;
    const unsigned long long k2l = r2 & (d.KB - 1), r3 = r2 >> d.log2KB;
    const unsigned long long u = r3 % d.U;
    const int g = (int)(r3 / d.U);
    const unsigned long long p = s * d.KB + k2l + d.L2 * (fs_p0(d, d.rank, g) / d.L2 + u);
    const unsigned long long k = fs_k_of_q(d, 2 * p + b) - (unsigned long long)d.rank * d.B;
    if (TO_BLOCK)
      dst[k] = src[e];
    else
      dst[e] = src[k];
  }
}

// transposed pack: h_t(k) = w_t(k) mult_k g_k (odd terms: odd k negated) at the
// slot pairs of this rank's k2 block, rows [t][k2l][k1] (read along k2l from
// the value exchange layout, written along k1)
__global__ void fs_tr_pack_kernel(FsDev d, const double* __restrict__ gx, const double* __restrict__ mult,
                                  int t0, int nt, BigTerms bt, const double2* __restrict__ wt,
                                  double2* __restrict__ rows, int* nonfinite) {
  __shared__ double2 tile[kFsTile][kFsTile + 1];
  constexpr int IT = kFsTile / kFsRows;
  const unsigned long long k10 = (unsigned long long)blockIdx.x * kFsTile;
  const unsigned long long k20 = (unsigned long long)blockIdx.y * kFsTile;
  const unsigned long long k2l = k20 + threadIdx.x;
  unsigned long long k0[IT];
  double gv[IT][2];
  bool ok[IT];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const unsigned long long k1 = k10 + threadIdx.y + kFsRows * it;
    ok[it] = k1 < d.L1 && k2l < d.KB;
    const unsigned long long p = (unsigned long long)d.rank * d.KB + k2l + d.L2 * k1;
    k0[it] = ok[it] ? fs_k_of_q(d, 2 * p) : 0;
    double2 pair = make_double2(0.0, 0.0);
    if (ok[it]) {
      const unsigned long long blk = k0[it] / d.B;
      pair = *reinterpret_cast<const double2*>(gx + fs_xpos(d, blk, blk, (int)(k0[it] & 1), k1, k2l));
      if (mult) {
        pair.x *= mult[k0[it]];
        pair.y *= mult[fs_k_of_q(d, 2 * p + 1)];
      }
    }
    gv[it][0] = pair.x;
    gv[it][1] = pair.y;
    if (nonfinite && t0 == 0 && ok[it] && (!isfinite(pair.x) || !isfinite(pair.y))) atomicOr(nonfinite, 1);
  }
  for (int t = 0; t < nt; ++t) {
    const int l = t0 + t;
    const int odd = big_odd(bt, l);
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const unsigned long long k1 = k10 + threadIdx.y + kFsRows * it;
      double2 h = make_double2(0.0, 0.0);
      if (ok[it]) {
        const double2 w = wt[((unsigned long long)l * d.L1 + k1) * d.KB + k2l];
        h = make_double2(w.x * gv[it][0], w.y * gv[it][1]);
        if (odd && (k0[it] & 1)) h = make_double2(-h.x, -h.y);
      }
      tile[threadIdx.x][threadIdx.y + kFsRows * it] = h;
    }
    __syncthreads();
    for (int ii = threadIdx.y; ii < kFsTile; ii += kFsRows) {  // write along k1
      const unsigned long long r = k20 + ii, k1 = k10 + threadIdx.x;
      if (r < d.KB && k1 < d.L1) rows[((unsigned long long)t * d.KB + r) * d.L1 + k1] = tile[ii][threadIdx.x];
    }
    __syncthreads();
  }
}

// rows [t][k2l][m1] (after the L1-point forward FFTs) times e^{-2 pi i m1 k2/L}
// into the exchange buffer (to the owner dest of m1: [t][i_dest][k2l])
__global__ void fs_tr_twiddle_kernel(FsDev d, const double2* __restrict__ rows, int nt,
                                     double2* __restrict__ send) {
  __shared__ double2 tile[kFsTile][kFsTile + 1];
  const int t = blockIdx.z;
  const unsigned long long m10 = (unsigned long long)blockIdx.x * kFsTile;
  const unsigned long long k0 = (unsigned long long)blockIdx.y * kFsTile;
  for (int kk = threadIdx.y; kk < kFsTile; kk += kFsRows) {  // read along m1
    const unsigned long long m1 = m10 + threadIdx.x, k2l = k0 + kk;
    double2 v = make_double2(0.0, 0.0);
    if (m1 < d.L1 && k2l < d.KB) {
      const unsigned long long k2 = (unsigned long long)d.rank * d.KB + k2l;
      double s, c;
      sincospi(-2.0 * (double)(m1 * k2) / (double)d.L, &s, &c);
      v = cmul(rows[((unsigned long long)t * d.KB + k2l) * d.L1 + m1], make_double2(c, s));
    }
    tile[threadIdx.x][kk] = v;
  }
  __syncthreads();
  for (int mm = threadIdx.y; mm < kFsTile; mm += kFsRows) {  // write along k2l
    const unsigned long long m1 = m10 + mm, k2l = k0 + threadIdx.x;
    if (m1 < d.L1 && k2l < d.KB) {
      const int dst = d.owner[m1];
      send[(unsigned long long)d.cum[dst] * d.KB * nt +
           ((unsigned long long)t * d.nres[dst] + d.lidx[m1]) * d.KB + k2l] = tile[mm][threadIdx.x];
    }
  }
}

// transposed unpack (big_tr_unpack_kernel's rows e = 0, 1): outputs r = a and
// r = L + a of a = res_i + L1 m2 from the packed entries a and L - a
__global__ void fs_tr_unpack_kernel(FsDev d, const double2* __restrict__ Z, int t0, int nt,
                                    BigTerms bt, double* __restrict__ chat, int first) {
  const unsigned long long J = 2 * d.L2;
  const unsigned long long total = (unsigned long long)d.nres_me * d.L2;
  const int* res_me = d.res_all + (size_t)d.rank * d.res_max;
  const double nd = (double)d.n;
  for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
       e += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long i = e >> d.log2L2, m2 = e & (d.L2 - 1);
    const unsigned long long res = (unsigned long long)res_me[i];
    const unsigned long long a = res + d.L1 * m2;
    unsigned long long ib, mb;
    if (res == 0) {
      ib = i;
      mb = (d.L2 - m2) & (d.L2 - 1);
    } else {
      ib = (unsigned long long)d.mirror[i];
      mb = d.L2 - 1 - m2;
    }
    const unsigned long long r[2] = {a, d.L + a};
    double c2[2], s2[2], ch[2], sh[2], acc[2] = {0.0, 0.0};
    double xr[2], ta[2], tb[2], tv[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      sincospi(-2.0 * (double)r[q] / nd, &s2[q], &c2[q]);
      sincospi((double)r[q] / (2.0 * nd), &sh[q], &ch[q]);
      xr[q] = (double)r[q] / nd;
      ta[q] = 1.0;
      tb[q] = xr[q];
    }
    for (int l = 0; l < t0 + nt; ++l) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (bt.cheb) {
          if (l == 0) {
            tv[q] = 1.0;
          } else if (l == 1) {
            tv[q] = xr[q];
          } else {
            const double nx = 2.0 * xr[q] * tb[q] - ta[q];
            ta[q] = tb[q];
            tb[q] = nx;
            tv[q] = nx;
          }
        } else {
          tv[q] = big_row(bt, l, xr[q]);
        }
      }
      if (l < t0) continue;
      const int tz = l - t0;
      const int odd = big_odd(bt, l);
      const double2 za = Z[((unsigned long long)tz * d.nres_me + i) * d.L2 + m2];
      const double2 zb = Z[((unsigned long long)tz * d.nres_me + ib) * d.L2 + mb];
      const double2 p0 = odd ? zb : za, p1 = odd ? za : zb;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        double x;
        if (!odd)
          x = big_tr_value(p0, p1, c2[q], s2[q], ch[q], sh[q]);
        else
          x = r[q] == 0 ? 0.0 : big_tr_value(p0, p1, c2[q], -s2[q], sh[q], ch[q]);
        acc[q] = __fma_rn(tv[q], x, acc[q]);
      }
    }
    double* o0 = chat + i * J + m2;
    double* o1 = chat + i * J + m2 + d.L2;
    *o0 = first ? acc[0] : *o0 + acc[0];
    *o1 = first ? acc[1] : *o1 + acc[1];
  }
}

unsigned fs_grid(unsigned long long total) {
  return (unsigned)std::min<unsigned long long>((total + 255) / 256, 8ull * sm_count() * 8);
}

BigTerms fs_terms(const FastNdct& p) {
  const bool cheb = p.bes_terms > 0;
  return BigTerms{0, 0, cheb ? 1 : 0, cheb ? p.swap : 0};
}

const double2* fs_weights(const FsLayout& f, const FastNdct& p, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(f.wt_mu);
  if (f.wt && f.wt_for == &p) return reinterpret_cast<const double2*>(f.wt);
  if (f.wt) {
    FLB_CUDA(cudaFree(f.wt));
    f.wt = nullptr;
  }
  const int terms = fast_ndct_terms(p);
  FLB_CUDA(cudaMalloc(&f.wt, (size_t)terms * f.B * sizeof(double)));
  ensure_recip();
  fs_weights_kernel<<<fs_grid(f.L1 * f.KB), 256, 0, s>>>(fs_dev(f), p.delta, terms, fs_terms(p),
                                                         reinterpret_cast<double2*>(f.wt));
  note_launch("fs_weights_kernel");
  f.wt_for = &p;
  return reinterpret_cast<const double2*>(f.wt);
}

void fs_check_terms(const FastNdct& p, const FsLayout& f, int t0, int t1) {
  if (p.n != f.n) fail(FL_INVALID_ARGUMENT, "four-step: layout and plan sizes differ");
  const int m = fast_ndct_terms(p);
  if (t0 < 0 || t1 > m || t0 >= t1) fail(FL_INVALID_ARGUMENT, "four-step: term range out of bounds");
}

}  // namespace

FsLayout* fs_create(size_t n, int world, int rank) {
  const int log2n = log2_exact(n);
  if (log2n < 0 || world < 1 || rank < 0 || rank >= world || (world & (world - 1)))
    fail(FL_INVALID_ARGUMENT, "four-step: N and the world size must be powers of two");
  const int log2L = log2n - 1;
  const int log2L1 = log2L / 2, log2L2 = log2L - log2L1;
  if (log2L2 > kMaxSmemLog2) fail(FL_INVALID_ARGUMENT, "four-step: N above 2^27");
  const size_t L1 = size_t(1) << log2L1, L2 = size_t(1) << log2L2;
  if (L1 < 2 * (size_t)world || L2 < (size_t)world)
    fail(FL_INVALID_ARGUMENT, "four-step: N too small for this world size (needs 2P <= L1)");
  auto* f = new FsLayout;
  f->n = n;
  f->L = n / 2;
  f->L1 = L1;
  f->L2 = L2;
  f->KB = L2 / world;
  f->B = n / world;
  f->U = L1 / (2 * world);
  f->log2n = log2n;
  f->log2L1 = log2L1;
  f->log2L2 = log2L2;
  f->log2KB = log2L2 - log2_exact((size_t)world);
  f->world = world;
  f->rank = rank;
  FLB_CUDA(cudaGetDevice(&f->device));
  // symmetric residue sets
  const size_t h = L1 / (2 * world);
  std::vector<std::vector<int>> res(world);
  for (int r = 0; r < world; ++r) {
    for (size_t j = r * h; j < (r + 1) * h; ++j) res[r].push_back((int)j);
    for (size_t j = r * h; j < (r + 1) * h; ++j)
      if (j != 0) res[r].push_back((int)(L1 - j));
    if (r == world - 1) res[r].push_back((int)(L1 / 2));
  }
  f->nres.resize(world);
  f->cum.assign(world + 1, 0);
  std::vector<int> owner(L1, -1), lidx(L1, -1);
  for (int r = 0; r < world; ++r) {
    f->nres[r] = (int)res[r].size();
    f->cum[r + 1] = f->cum[r] + f->nres[r];
    f->res_max = std::max(f->res_max, res[r].size());
    for (size_t i = 0; i < res[r].size(); ++i) {
      owner[res[r][i]] = r;
      lidx[res[r][i]] = (int)i;
    }
  }
  std::vector<int> all((size_t)world * f->res_max, -1);
  for (int r = 0; r < world; ++r)
    std::copy(res[r].begin(), res[r].end(), all.begin() + (size_t)r * f->res_max);
  std::vector<int> mirror(res[rank].size());
  for (size_t i = 0; i < res[rank].size(); ++i) mirror[i] = lidx[(L1 - res[rank][i]) % L1];
  auto up = [](const std::vector<int>& v, int** dst) {
    FLB_CUDA(cudaMalloc(dst, std::max<size_t>(1, v.size()) * sizeof(int)));
    FLB_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
  };
  try {
    up(all, &f->d_res_all);
    up(mirror, &f->d_mirror);
    up(owner, &f->d_owner);
    up(lidx, &f->d_lidx);
    up(f->cum, &f->d_cum);
    up(f->nres, &f->d_nres);
  } catch (...) {
    fs_destroy(f);
    throw;
  }
  return f;
}

void fs_destroy(FsLayout* f) {
  if (!f) return;
  for (int* q : {f->d_res_all, f->d_mirror, f->d_owner, f->d_lidx, f->d_cum, f->d_nres})
    if (q) cudaFree(q);
  if (f->wt) cudaFree(f->wt);
  delete f;
}

FsInfo fs_info(const FsLayout& f) {
  return FsInfo{f.n, f.L, f.L1, f.L2, f.KB, f.B, (size_t)f.nres[f.rank], f.res_max, f.world, f.rank};
}

size_t fs_coef_count(const FsLayout& f, int transpose, int peer, int send) {
  if (peer < 0 || peer >= f.world) fail(FL_INVALID_ARGUMENT, "four-step: peer out of range");
  // forward: sender's residues; transpose: receiver's residues
  const bool mine = transpose ? !send : send;
  return (size_t)(mine ? f.nres[f.rank] : f.nres[peer]) * f.KB;
}

void fs_to_residue(const FsLayout& f, const double* full, double* send, cudaStream_t s) {
  const FsDev d = fs_dev(f);
  const dim3 grid((unsigned)((2 * f.L2 + kFsTile - 1) / kFsTile),
                  (unsigned)((f.res_max + kFsTile - 1) / kFsTile), (unsigned)f.world);
  fs_residue_kernel<true><<<grid, dim3(kFsTile, kFsRows), 0, s>>>(d, full, send);
  note_launch("fs_residue_kernel");
}

void fs_from_residue(const FsLayout& f, const double* gathered, double* full, cudaStream_t s) {
  const FsDev d = fs_dev(f);
  const dim3 grid((unsigned)((2 * f.L2 + kFsTile - 1) / kFsTile),
                  (unsigned)((f.res_max + kFsTile - 1) / kFsTile), (unsigned)f.world);
  fs_residue_kernel<false><<<grid, dim3(kFsTile, kFsRows), 0, s>>>(d, gathered, full);
  note_launch("fs_residue_kernel");
}

void fs_fwd1(const FsLayout& f, const FastNdct& p, int t0, int t1, const double* chat,
             double2* send, double2* work, int* nonfinite, cudaStream_t s) {
  fs_check_terms(p, f, t0, t1);
  const FsDev d = fs_dev(f);
  const int nt = t1 - t0;
  ensure_recip();
  const unsigned long long items = (unsigned long long)d.nres_me * f.L2;
  fs_fwd_pack_kernel<<<fs_grid(items), 256, 0, s>>>(d, chat, t0, nt, fs_terms(p), work, nonfinite);
  note_launch("fs_fwd_pack_kernel");
  fft_pow2(work, nullptr, f.log2L2, (size_t)nt * d.nres_me, true, s);
  fs_fwd_twiddle_kernel<<<fs_grid(items * nt), 256, 0, s>>>(d, work, nt, send);
  note_launch("fs_fwd_twiddle_kernel");
}

void fs_fwd2(const FsLayout& f, const FastNdct& p, int t0, int t1, const double2* recv,
             double2* work, double* fx, int first, cudaStream_t s) {
  fs_check_terms(p, f, t0, t1);
  const FsDev d = fs_dev(f);
  const int nt = t1 - t0;
  ensure_recip();
  const dim3 tb(kFsTile, kFsRows);
  const unsigned gx = (unsigned)((f.L1 + kFsTile - 1) / kFsTile), gy = (unsigned)((f.KB + kFsTile - 1) / kFsTile);
  fs_fwd_gather_kernel<<<dim3(gx, gy, (unsigned)nt), tb, 0, s>>>(d, recv, nt, work);
  note_launch("fs_fwd_gather_kernel");
  fft_pow2(work, nullptr, f.log2L1, (size_t)nt * f.KB, true, s);
  const double2* wt = fs_weights(f, p, s);
  fs_fwd_unpack_kernel<<<dim3(gx, gy), tb, 0, s>>>(d, work, t0, nt, fs_terms(p), wt, fx, first);
  note_launch("fs_fwd_unpack_kernel");
}

void fs_values_from_exchange(const FsLayout& f, const double* fx, double* block, cudaStream_t s) {
  fs_values_kernel<true><<<fs_grid(f.B), 256, 0, s>>>(fs_dev(f), fx, block);
  note_launch("fs_values_kernel");
}

void fs_values_to_exchange(const FsLayout& f, const double* block, double* fx, cudaStream_t s) {
  fs_values_kernel<false><<<fs_grid(f.B), 256, 0, s>>>(fs_dev(f), block, fx);
  note_launch("fs_values_kernel");
}

void fs_tr1(const FsLayout& f, const FastNdct& p, const double* mult, int t0, int t1,
            const double* gx, double2* send, double2* work, int* nonfinite, cudaStream_t s) {
  fs_check_terms(p, f, t0, t1);
  const FsDev d = fs_dev(f);
  const int nt = t1 - t0;
  ensure_recip();
  const dim3 tb(kFsTile, kFsRows);
  const unsigned gx1 = (unsigned)((f.L1 + kFsTile - 1) / kFsTile), gy = (unsigned)((f.KB + kFsTile - 1) / kFsTile);
  const double2* wt = fs_weights(f, p, s);
  fs_tr_pack_kernel<<<dim3(gx1, gy), tb, 0, s>>>(d, gx, mult, t0, nt, fs_terms(p), wt, work, nonfinite);
  note_launch("fs_tr_pack_kernel");
  fft_pow2(work, nullptr, f.log2L1, (size_t)nt * f.KB, false, s);
  fs_tr_twiddle_kernel<<<dim3(gx1, gy, (unsigned)nt), tb, 0, s>>>(d, work, nt, send);
  note_launch("fs_tr_twiddle_kernel");
}

void fs_tr2(const FsLayout& f, const FastNdct& p, int t0, int t1, const double2* recv,
            double2* work, double* chat, int first, cudaStream_t s) {
  fs_check_terms(p, f, t0, t1);
  const FsDev d = fs_dev(f);
  const int nt = t1 - t0;
  // [src][t][i][k2l] -> rows [t][i][k2 = src KB + k2l]
  const size_t chunk = (size_t)nt * d.nres_me * f.KB;
  for (int src = 0; src < f.world; ++src)
    FLB_CUDA(cudaMemcpy2DAsync(work + (size_t)src * f.KB, f.L2 * sizeof(double2), recv + src * chunk,
                               f.KB * sizeof(double2), f.KB * sizeof(double2), (size_t)nt * d.nres_me,
                               cudaMemcpyDeviceToDevice, s));
  fft_pow2(work, nullptr, f.log2L2, (size_t)nt * d.nres_me, false, s);
  const unsigned long long items = (unsigned long long)d.nres_me * f.L2;
  fs_tr_unpack_kernel<<<fs_grid(items), 256, 0, s>>>(d, work, t0, nt, fs_terms(p), chat, first);
  note_launch("fs_tr_unpack_kernel");
}

}  // namespace flb
