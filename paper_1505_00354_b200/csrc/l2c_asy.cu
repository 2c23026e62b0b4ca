// Asymptotic-expansion Legendre <-> Chebyshev conversion (see l2c_asy.cuh).
//
// Reference: conversion.hpp:100-118 (leg2cheb_apply) and :121-140 (the
// transpose) compute the same products by their O(N^2) loops; PAPER.md
// cites Hale & Townsend's asymptotic method as the fast one. The algorithm
// restated (tools/asy_model.py checks a NumPy version of it against the
// oracle):
//
//   P_n(cos t) = C_n sum_{m<M} h_{m,n} cos((n+m+1/2) t - (m+1/2) pi/2) / (2 sin t)^{m+1/2} + R,
//   C_n = (4/pi) prod_{j<=n} j/(j+1/2) = 2 / (pi (n+1/2) s_n),
//   h_{m,n} = prod_{j<=m} (j-1/2)^2 / (j (n+j+1/2)),  |R| <= C_n h_{M,n} 2/(2 sin t)^{M+1/2}.
//
// Levels nu_0 < nu_1 < ... (ratio R): at level l the expansion is used for
// the degrees n >= nu_l at the points with sin t >= S_l (R <= 2^-54 there).
// Per level and term m, cos((n+m+1/2)t - (m+1/2)pi/2) = Re(e^{i n t} g_m(t)),
// g_m(t) = e^{i (m+1/2)(t - pi/2)}, so the level's contribution at t_k is
//   sum_m Re(g_m(t_k)) DCT3[u_m](k) - Im(g_m(t_k)) DST3[u_m](k) / (2 sin t_k)^{m+1/2},
//   u_{m,n} = c_n C_n h_{m,n} [n >= nu_l]:
// 2M real transforms per level, all of them in one batched multi-pass FFT
// (the NDCT's Makhoul packing, fft_pow2), the output weights applied in the
// unpack only at the level's points. The degrees below a point's cutoff
// (all N for the few points nearest the ends) come from the recurrence in
// y = 2 sin^2(t/2): d_{n+1} = (n d_n - (2n+1) y P_n)/(n+1), P_{n+1} = P_n + d_{n+1},
// evaluated for the point pair (k, N-1-k) at once (P_n(-x) = (-1)^n P_n(x)).
// Long chains are cut into chunks: per chunk a 2x2 transfer matrix (two basis
// runs), a short sequential prefix over the chunks, then every chunk again
// from its true start state -- all chunks in parallel.
#include "l2c_asy.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "fast_ndct.cuh"
#include "fft.cuh"
#include "launch.cuh"

namespace flb {
namespace {

constexpr int kMaxLev = 24;
constexpr int kMaxM = 24;
constexpr int kMaxBands = kMaxLev + 1;
constexpr int kPairsPerWarp = 64;  // two pairs per lane: p = p0 + 64 g + 32 i + lane
constexpr int kRecThreads = 128;
// pairs per lane in the transposed recurrence (summed in the lane before the
// cross-lane reduction): super-groups of 32 kTrPairs pairs
#ifndef FLB_ASY_TR_PAIRS
#define FLB_ASY_TR_PAIRS 4
#endif
constexpr int kTrPairs = FLB_ASY_TR_PAIRS;
constexpr int kTrGroups = kTrPairs / 2;  // groups of 64 pairs per super-group

// The expansion's levels, by pair index (kernel parameter).
struct LevTab {
  int L, M;
  long long nu[kMaxLev];      // level l: degrees n >= nu[l] (increasing in l)
  long long pb[kMaxLev + 1];  // level l owns pairs [pb[l+1], pb[l]); pb[0] = N/2;
                              // pairs below pb[L] have no level (recurrence to N)
  double hk[kMaxM];           // (t - 1/2)^2 / t, t >= 1
};

__device__ __forceinline__ int level_of(const LevTab& t, long long pk) {
  int l = 0;
  while (l < t.L && pk < t.pb[l + 1]) ++l;
  return l;
}

// Recurrence bands: pairs [p0, p1) summing the degrees [0, nu).
struct RecBand {
  long long p0, p1, nu;
  int lc, Q, G, W;     // chunk length, chunks, groups of 64 pairs, transposed workers per chunk
  long long wbase;     // warps (g, q): wbase + g Q + q          (transfer, forward)
  long long xbase;     // transposed worker warps (q, w): xbase + q W + w
  long long ibase;     // per-(g, q) pair slots: ibase + (g Q + q) 64 + 32 i + lane
  long long gbase;     // pair slots g 64 + 32 i + lane (prefix kernel threads)
  long long rbase;     // transposed partial rows: rbase + (q W + w) lc + offset
};
struct RecTab {
  int nb;
  long long nwarps, nxwarps, nslots, ngslots, nrows;
  RecBand b[kMaxBands];
};

__device__ __forceinline__ int band_of_warp(const RecTab& t, long long w) {
  int b = 0;
  while (b + 1 < t.nb && w >= t.b[b + 1].wbase) ++b;
  return b;
}

// y = 2 sin^2(t_p / 2) = 1 - cos t_p, t_p = (p + 1/2) pi / N (exact argument)
__device__ __forceinline__ double pair_y(long long p, double nd) {
  const double s = sinpi((2.0 * (double)p + 1.0) / (4.0 * nd));
  return 2.0 * s * s;
}

// One step S_n -> S_{n+1} of the recurrence, (a, b) = (n/(n+1), (2n+1)/(n+1)).
__device__ __forceinline__ void rec_step(double2 ab, double y, double& P, double& d) {
  const double by = ab.y * y;
  d = __fma_rn(-by, P, ab.x * d);
  P += d;
}

// The same step carrying Q = y P instead of P (the forward chains: four FP64
// instructions per step instead of five -- a d, the fused update of d, the
// fused update of Q, and the caller's weighted sum; sums of c_n Q_n are
// divided by y once at the end).
__device__ __forceinline__ void rec_step_q(double2 ab, double y, double& Q, double& d) {
  d = __fma_rn(-ab.y, Q, ab.x * d);
  Q = __fma_rn(y, d, Q);
}

// Per-warp shared-memory ring of the recurrence coefficients (and the forward
// kernel's inputs), 32 steps per slot, filled by cp.async kAhead windows ahead
// of use: the chains are latency-bound, and an L2 load per step (or a
// register prefetch one block ahead) stalls every step for the load latency.
constexpr int kRing = 8, kAhead = 6;
struct WarpRing {
  double2 ab[kRing][32];
  double c[kRing][32];
};
__device__ __forceinline__ void cp_async(void* sdst, const void* gsrc, int bytes, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  if (bytes == 16)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gsrc), "r"(valid ? 16 : 0)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gsrc), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_ahead() {
  asm volatile("cp.async.wait_group %0;" ::"n"(kAhead - 1) : "memory");
}
// window k (steps w0 = base + 32 k + lane) into its ring slot; one commit group
__device__ __forceinline__ void ring_issue(WarpRing& r, const double2* __restrict__ ab,
                                           const double* __restrict__ c, long long base, long long k,
                                           long long end, int lane) {
  // (windows past the end issue nothing, so no copy is left in flight after the
  // last window: the next super-group's prologue may reuse every slot)
  const long long w0 = base + 32 * k, nn = w0 + lane;
  if (w0 < end) {
    const bool ok = nn < end;
    const int slot = (int)(k % kRing);
    cp_async(&r.ab[slot][lane], ok ? ab + nn : ab, 16, ok);
    if (c) cp_async(&r.c[slot][lane], ok ? c + nn : c, 8, ok);
  }
  cp_commit();
}

// ---- plan-time tables -------------------------------------------------------
__global__ void asy_tables_kernel(long long n, const double* __restrict__ s, double* __restrict__ Cn,
                                  double2* __restrict__ ab) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double jd = (double)j;
  Cn[j] = 2.0 / (kPi * (jd + 0.5) * s[j]);
  ab[j] = make_double2(jd / (jd + 1.0), (2.0 * jd + 1.0) / (jd + 1.0));
}

// ---- recurrence: transfer matrices of the chunks ---------------------------
// Chunk q < Q - 1 maps S_{q lc} (q = 0: S_1) to S_{(q+1) lc}: the images of
// (1, 0) and (0, 1) under its steps.
__global__ void __launch_bounds__(kRecThreads) asy_rec_transfer_kernel(
    const __grid_constant__ RecTab t, const double2* __restrict__ ab, double nd, double4* __restrict__ T) {
  __shared__ WarpRing rings[kRecThreads / 32];
  const long long w = (blockIdx.x * (long long)kRecThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= t.nwarps) return;
  WarpRing& rg = rings[threadIdx.x >> 5];
  const RecBand& B = t.b[band_of_warp(t, w)];
  const long long loc = w - B.wbase, g = loc / B.Q;
  const int q = (int)(loc % B.Q);
  if (q == B.Q - 1) return;
  const long long base = (long long)q * B.lc, end = base + B.lc;
  double y[2], PA[2], dA[2], PB[2], dB[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const long long p = B.p0 + g * kPairsPerWarp + 32 * i + lane;
    y[i] = p < B.p1 ? pair_y(p, nd) : 0.0;
    PA[i] = 1.0;
    dA[i] = 0.0;
    PB[i] = 0.0;
    dB[i] = 1.0;
  }
  const long long nw = B.lc / 32;
  for (int k = 0; k < kAhead; ++k) ring_issue(rg, ab, nullptr, base, k, end, lane);
  for (long long k = 0; k < nw; ++k) {
    cp_wait_ahead();
    __syncwarp();
    const double2* A = rg.ab[k % kRing];
    // straight-line 32 steps (no per-step branch: the shared-memory loads are
    // hoisted ahead of the dependent chain); the first window of q = 0 starts at S_1
    const int j0 = base + 32 * k == 0 ? 1 : 0;
    if (j0 == 0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double2 cf = A[j];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          rec_step(cf, y[i], PA[i], dA[i]);
          rec_step(cf, y[i], PB[i], dB[i]);
        }
      }
    } else {
      for (int j = 1; j < 32; ++j) {
        const double2 cf = A[j];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          rec_step(cf, y[i], PA[i], dA[i]);
          rec_step(cf, y[i], PB[i], dB[i]);
        }
      }
    }
    __syncwarp();
    ring_issue(rg, ab, nullptr, base, k + kAhead, end, lane);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const long long p = B.p0 + g * kPairsPerWarp + 32 * i + lane;
    if (p < B.p1) T[B.ibase + loc * kPairsPerWarp + 32 * i + lane] = make_double4(PA[i], dA[i], PB[i], dB[i]);
  }
}

// ---- recurrence: chunk start states (sequential over the chunks of a pair) ---
__global__ void asy_rec_prefix_kernel(const __grid_constant__ RecTab t, const double4* __restrict__ T,
                                      double2* __restrict__ St, double nd) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= t.ngslots) return;
  int b = 0;
  while (b + 1 < t.nb && i >= t.b[b + 1].gbase) ++b;
  const RecBand& B = t.b[b];
  if (B.Q < 2) return;
  const long long loc = i - B.gbase, g = loc / kPairsPerWarp, slot = loc % kPairsPerWarp;
  const long long p = B.p0 + loc;
  if (p >= B.p1) return;
  const double y = pair_y(p, nd);
  double P = 1.0 - y, d = -y;  // S_1
  const long long base = B.ibase + g * (long long)B.Q * kPairsPerWarp + slot;
  for (int q = 0; q + 1 < B.Q; ++q) {
    const double4 m = T[base + (long long)q * kPairsPerWarp];
    const double P2 = __fma_rn(P, m.x, d * m.z);
    d = __fma_rn(P, m.y, d * m.w);
    P = P2;
    St[base + (long long)(q + 1) * kPairsPerWarp] = make_double2(P, d);
  }
}

// ---- recurrence, forward: per (pair, chunk) partial sums of even / odd degrees
__global__ void __launch_bounds__(kRecThreads) asy_rec_fwd_kernel(
    const __grid_constant__ RecTab t, const double2* __restrict__ ab, const double* __restrict__ c, size_t ld,
    const double2* __restrict__ St, double2* __restrict__ Ep, double nd) {
  __shared__ WarpRing rings[kRecThreads / 32];
  const long long w = (blockIdx.x * (long long)kRecThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= t.nwarps) return;
  WarpRing& rg = rings[threadIdx.x >> 5];
  const size_t col = blockIdx.y;
  c += col * ld;
  Ep += col * t.nslots;
  const RecBand& B = t.b[band_of_warp(t, w)];
  const long long loc = w - B.wbase, g = loc / B.Q;
  const int q = (int)(loc % B.Q);
  const long long base = (long long)q * B.lc;
  const long long end = min(base + B.lc, B.nu);
  double y[2], P[2], d[2], E[2], O[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const long long p = B.p0 + g * kPairsPerWarp + 32 * i + lane;
    const bool ok = p < B.p1;
    y[i] = ok ? pair_y(p, nd) : 0.0;
    if (q == 0) {
      P[i] = 1.0 - y[i];
      d[i] = -y[i];
    } else {
      const double2 s0 = ok ? St[B.ibase + loc * kPairsPerWarp + 32 * i + lane] : make_double2(0.0, 0.0);
      P[i] = s0.x;
      d[i] = s0.y;
    }
    P[i] *= y[i];  // the chain carries Q = y P
    E[i] = 0.0;
    O[i] = 0.0;
  }
  const long long nw = (end - base + 31) / 32;
  for (int k = 0; k < kAhead; ++k) ring_issue(rg, ab, c, base, k, end, lane);
  for (long long k = 0; k < nw; ++k) {
    cp_wait_ahead();
    __syncwarp();
    const int slot = (int)(k % kRing);
    const long long w0 = base + 32 * k;
    if (w0 + 32 <= end && w0 > 0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double2 cf = rg.ab[slot][j];
        const double cn = rg.c[slot][j];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (j & 1)
            O[i] = __fma_rn(cn, P[i], O[i]);
          else
            E[i] = __fma_rn(cn, P[i], E[i]);
          rec_step_q(cf, y[i], P[i], d[i]);
        }
      }
    } else {
      for (int j = 0; j < 32 && w0 + j < end; ++j) {
        const double cn = rg.c[slot][j];
        if (w0 + j == 0) {  // P_0 = 1; the state already holds S_1
#pragma unroll
          for (int i = 0; i < 2; ++i) E[i] = __fma_rn(cn, y[i], E[i]);
          continue;
        }
        const double2 cf = rg.ab[slot][j];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (j & 1)
            O[i] = __fma_rn(cn, P[i], O[i]);
          else
            E[i] = __fma_rn(cn, P[i], E[i]);
          rec_step_q(cf, y[i], P[i], d[i]);
        }
      }
    }
    __syncwarp();
    ring_issue(rg, ab, c, base, k + kAhead, end, lane);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const long long p = B.p0 + g * kPairsPerWarp + 32 * i + lane;
    if (p < B.p1)  // sums of c_n y P_n: back to sums of c_n P_n
      Ep[B.ibase + loc * kPairsPerWarp + 32 * i + lane] = make_double2(E[i] / y[i], O[i] / y[i]);
  }
}

// f_k += E + O, f_{N-1-k} += E - O (F zeroed; the expansion levels add to it too)
__global__ void asy_rec_fwd_finish_kernel(const __grid_constant__ RecTab t, const double2* __restrict__ Ep,
                                          double* __restrict__ F, size_t ldF, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= t.ngslots) return;
  const size_t col = blockIdx.y;
  Ep += col * t.nslots;
  F += col * ldF;
  int b = 0;
  while (b + 1 < t.nb && i >= t.b[b + 1].gbase) ++b;
  const RecBand& B = t.b[b];
  const long long loc = i - B.gbase, g = loc / kPairsPerWarp, slot = loc % kPairsPerWarp;
  const long long p = B.p0 + loc;
  if (p >= B.p1) return;
  const long long base = B.ibase + g * (long long)B.Q * kPairsPerWarp + slot;
  double E = 0.0, O = 0.0;
  for (int q = 0; q < B.Q; ++q) {
    const double2 v = Ep[base + (long long)q * kPairsPerWarp];
    E += v.x;
    O += v.y;
  }
  F[p] += E + O;
  F[n - 1 - p] += E - O;
}

// lane i gets sum over the warp's lanes of v[i] (31 shuffles, recursive halving)
__device__ __forceinline__ double warp_transpose_sum(double (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < s; ++j) {
      const double send = up ? v[j] : v[j + s];
      const double keep = up ? v[j + s] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// ---- recurrence, transpose: out_n += sum_k P_n(x_k) f_k over the points whose
// cutoff exceeds n. Worker (q, w) of a band runs the super-groups gg = w,
// w + W, ... (128 pairs: groups 2gg, 2gg + 1, four pairs per lane, summed in
// the lane before the cross-lane reduction) over chunk q; per 32-degree window
// the lanes' values are summed across the warp and accumulated into the
// worker's private row of R (the first super-group writes it).
__global__ void __launch_bounds__(kRecThreads) asy_rec_tr_kernel(
    const __grid_constant__ RecTab t, const double2* __restrict__ ab, const double* __restrict__ F,
    size_t ldF, const double2* __restrict__ St, double* __restrict__ R, double nd, long long n) {
  __shared__ WarpRing rings[kRecThreads / 32];
  const long long w = (blockIdx.x * (long long)kRecThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= t.nxwarps) return;
  WarpRing& rg = rings[threadIdx.x >> 5];
  const size_t col = blockIdx.y;
  F += col * ldF;
  R += col * t.nrows;
  int b = 0;
  while (b + 1 < t.nb && w >= t.b[b + 1].xbase) ++b;
  const RecBand& B = t.b[b];
  const long long loc = w - B.xbase;
  const int q = (int)(loc / B.W), wk = (int)(loc % B.W);
  const long long start = (long long)q * B.lc;
  const long long end = min((long long)(q + 1) * B.lc, B.nu);
  const long long G2 = (B.G + kTrGroups - 1) / kTrGroups;
  double* row = R + B.rbase + ((long long)q * B.W + wk) * B.lc;
  for (long long gg = wk; gg < G2; gg += B.W) {
    double y[kTrPairs], P[kTrPairs], d[kTrPairs], ue[kTrPairs], uo[kTrPairs];
#pragma unroll
    for (int i = 0; i < kTrPairs; ++i) {
      const long long g = kTrGroups * gg + (i >> 1);
      const long long p = B.p0 + g * kPairsPerWarp + 32 * (i & 1) + lane;
      const bool ok = p < B.p1;
      y[i] = ok ? pair_y(p, nd) : 0.0;
      const double fp = ok ? F[p] : 0.0, fm = ok ? F[n - 1 - p] : 0.0;
      ue[i] = fp + fm;
      uo[i] = fp - fm;
      if (q == 0) {
        P[i] = 1.0 - y[i];
        d[i] = -y[i];
      } else {
        const double2 s0 = ok ? St[B.ibase + (g * B.Q + q) * kPairsPerWarp + 32 * (i & 1) + lane]
                              : make_double2(0.0, 0.0);
        P[i] = s0.x;
        d[i] = s0.y;
      }
    }
    const long long nw = (end - start + 31) / 32;
    for (int k = 0; k < kAhead; ++k) ring_issue(rg, ab, nullptr, start, k, end, lane);
    for (long long k = 0; k < nw; ++k) {
      const long long w0 = start + 32 * k;
      cp_wait_ahead();
      __syncwarp();
      const double2* A = rg.ab[k % kRing];
      double v[32];
      if (w0 > 0 && w0 + 32 <= end) {  // straight-line window (see the transfer kernel)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const double2 cf = A[j];
          double val = 0.0;
#pragma unroll
          for (int i = 0; i < kTrPairs; ++i) {
            val = __fma_rn(P[i], (j & 1) ? uo[i] : ue[i], val);
            rec_step(cf, y[i], P[i], d[i]);
          }
          v[j] = val;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const long long nn = w0 + j;
          double val = 0.0;
          if (nn < end) {
            if (nn == 0) {
#pragma unroll
              for (int i = 0; i < kTrPairs; ++i) val += ue[i];  // P_0 = 1; the state holds S_1
            } else {
              const double2 cf = A[j];
#pragma unroll
              for (int i = 0; i < kTrPairs; ++i) {
                val = __fma_rn(P[i], (j & 1) ? uo[i] : ue[i], val);
                rec_step(cf, y[i], P[i], d[i]);
              }
            }
          }
          v[j] = val;
        }
      }
      __syncwarp();
      ring_issue(rg, ab, nullptr, start, k + kAhead, end, lane);
      const double sum = warp_transpose_sum(v, lane);
      const long long o = w0 - start + lane;
      if (w0 + lane < end) row[o] = gg == wk ? sum : row[o] + sum;
    }
  }
}

// out_n = (out_n + sum over bands / workers of R) * ((n + 1/2) if scale_half)
__global__ void __launch_bounds__(256) asy_rec_tr_finish_kernel(const __grid_constant__ RecTab t, const double* __restrict__ R,
                                                                double* __restrict__ out, size_t ld,
                                                                long long n, int scale_half) {
  __shared__ double part[8][32];
  const size_t col = blockIdx.y;
  R += col * t.nrows;
  const long long n0 = (long long)blockIdx.x * 32;
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const long long r = n0 + lane;
  double acc = 0.0;
  for (int b = 0; b < t.nb; ++b) {
    const RecBand& B = t.b[b];
    if (B.nu <= n0 || B.G == 0) continue;
    const long long q = n0 / B.lc, off = n0 - q * B.lc + lane;
    if (r >= B.nu) continue;
    for (int w = wi; w < B.W; w += 8) acc += R[B.rbase + (q * B.W + w) * B.lc + off];
  }
  part[wi][lane] = acc;
  __syncthreads();
  if (wi == 0 && r < n) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += part[k][lane];
    double* o = out + col * ld + r;
    const double v = *o + s;
    *o = scale_half ? v * ((double)r + 0.5) : v;
  }
}

// ---- expansion levels: forward pack (u_{m,n} of every level of the batch and
// every term, DCT-III and DST-III packing into N/2-point complex rows) --------
__global__ void __launch_bounds__(256) asy_fwd_pack_kernel(const __grid_constant__ LevTab lt, int l0, int m0,
                                                           int nm, const double* __restrict__ c,
                                                           size_t ld, const double* __restrict__ Cn,
                                                           long long n, size_t nc,
                                                           double2* __restrict__ Z) {
  const long long P = n / 2;
  const size_t col = blockIdx.y;
  const int lv = blockIdx.z;
  const long long nu = lt.nu[l0 + lv];
  const double* cc = c + col * ld;
  const double nd = (double)n;
  for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < P;
       m += (long long)gridDim.x * blockDim.x) {
    const long long js[4] = {m, n - m, m + P, P - m};
    double bs[4], h[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const long long j = js[r];
      bs[r] = (j < n && j >= nu) ? __ldg(cc + j) * __ldg(Cn + j) : 0.0;
      h[r] = 1.0;
    }
    double sa, ca, sb, cb, s4, c4;
    sincospi((double)m / (2.0 * nd), &sa, &ca);
    sincospi((double)(m + P) / (2.0 * nd), &sb, &cb);
    sincospi(2.0 * (double)m / nd, &s4, &c4);
    auto emit = [&](double xa, double xan, double xb, double xbn) {
      const double2 Wa = make_double2(ca * xa + sa * xan, sa * xa - ca * xan);
      const double2 Wb = make_double2(cb * xb + sb * xbn, sb * xb - cb * xbn);
      const double2 sm = make_double2(Wa.x + Wb.x, Wa.y + Wb.y);
      const double2 dd2 = make_double2(Wa.x - Wb.x, Wa.y - Wb.y);
      const double2 dr = make_double2(dd2.x * c4 - dd2.y * s4, dd2.x * s4 + dd2.y * c4);
      return make_double2(sm.x - dr.y, sm.y + dr.x);
    };
    for (int tm = 0; tm < m0 + nm; ++tm) {
      if (tm > 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) h[r] = h[r] * lt.hk[tm] * __drcp_rn((double)js[r] + (double)tm + 0.5);
      }
      if (tm < m0) continue;
      const double st0 = bs[0] * h[0], st1 = bs[1] * h[1], st2 = bs[2] * h[2], st3 = bs[3] * h[3];
      // DCT-III: X(0) = st(0), X(j) = st(j)/2; DST-III: X(0) = 0, X(j) = st(N - j)/2
      const double2 zc = emit(m == 0 ? st0 : 0.5 * st0, m == 0 ? 0.0 : 0.5 * st1, 0.5 * st2, 0.5 * st3);
      const double2 zs = emit(m == 0 ? 0.0 : 0.5 * st1, m == 0 ? 0.0 : 0.5 * st0, 0.5 * st3, 0.5 * st2);
      const size_t tr = ((size_t)(lv * nm + tm - m0) * 2) * nc + col;
      Z[tr * P + m] = zc;
      Z[(tr + nc) * P + m] = zs;
    }
  }
}

// e^{i (t_k - pi/2)/2} / sqrt(2 sin t_k) and the ratio e^{i (t_k - pi/2)} / (2 sin t_k)
__device__ __forceinline__ void asy_weights(long long k, long long pk, double nd, double2& g,
                                            double2& rho) {
  const double s2 = 2.0 * sinpi((2.0 * (double)pk + 1.0) / (2.0 * nd));
  double sh, chh, s1, c1;
  const double num = 2.0 * (double)k + 1.0 - nd;
  sincospi(num / (4.0 * nd), &sh, &chh);
  sincospi(num / (2.0 * nd), &s1, &c1);
  const double r = 1.0 / sqrt(s2);
  g = make_double2(chh * r, sh * r);
  const double q = 1.0 / s2;
  rho = make_double2(c1 * q, s1 * q);
}

// ---- expansion levels: forward unpack at the points of the batch's levels ---
__global__ void __launch_bounds__(256) asy_fwd_unpack_kernel(const __grid_constant__ LevTab lt, int l0, int l1,
                                                             int m0, int nm,
                                                             const double2* __restrict__ Z, long long n,
                                                             size_t nc, double* __restrict__ F,
                                                             size_t ldF) {
  const long long P = n / 2;
  const size_t col = blockIdx.y;
  const long long lo = lt.pb[l1], hi = lt.pb[l0], cnt = hi - lo;
  const double nd = (double)n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < 2 * cnt;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long k = idx < cnt ? lo + idx : n - 1 - (lo + idx - cnt);
    const long long pk = min(k, n - 1 - k);
    const int lv = level_of(lt, pk) - l0;
    const long long qq = (k & 1) ? n - 1 - (k >> 1) : (k >> 1);
    const long long qi = qq >> 1;
    const bool comp = qq & 1;
    const double sgn = (k & 1) ? -1.0 : 1.0;
    double2 g, rho;
    asy_weights(k, pk, nd, g, rho);
    for (int tm = 0; tm < m0; ++tm) g = cmul(g, rho);
    double acc = 0.0;
    for (int tm = 0; tm < nm; ++tm) {
      const size_t tr = ((size_t)(lv * nm + tm) * 2) * nc + col;
      const double2 zc = Z[tr * P + qi], zs = Z[(tr + nc) * P + qi];
      const double yc = comp ? zc.y : zc.x;
      const double ys = sgn * (comp ? zs.y : zs.x);
      acc += g.x * yc - g.y * ys;
      g = cmul(g, rho);
    }
    F[col * ldF + k] += acc;
  }
}

// ---- expansion levels: transposed pack (weighted values of the level's points)
__global__ void __launch_bounds__(256) asy_tr_pack_kernel(const __grid_constant__ LevTab lt, int l0, int m0,
                                                          int nm, const double* __restrict__ F,
                                                          size_t ldF, long long n, size_t nc,
                                                          double2* __restrict__ Z) {
  const long long P = n / 2;
  const size_t col = blockIdx.y;
  const int lv = blockIdx.z, l = l0 + lv;
  const double nd = (double)n;
  const double* f = F + col * ldF;
  for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < P;
       m += (long long)gridDim.x * blockDim.x) {
    long long ks[2];
    double fv[2];
    double2 g[2], rho[2];
    bool any = false;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const long long q = 2 * m + e;
      const long long k = q < P ? 2 * q : 2 * (n - 1 - q) + 1;
      ks[e] = k;
      const long long pk = min(k, n - 1 - k);
      const bool in = level_of(lt, pk) == l;
      fv[e] = in ? f[k] : 0.0;
      any |= in;
      if (in) {
        asy_weights(k, pk, nd, g[e], rho[e]);
        for (int tm = 0; tm < m0; ++tm) g[e] = cmul(g[e], rho[e]);
      } else {
        g[e] = make_double2(0.0, 0.0);
        rho[e] = make_double2(0.0, 0.0);
      }
    }
    const double s0 = (ks[0] & 1) ? -1.0 : 1.0, s1 = (ks[1] & 1) ? -1.0 : 1.0;
    for (int tm = 0; tm < nm; ++tm) {
      const size_t tr = ((size_t)(lv * nm + tm) * 2) * nc + col;
      double2 zc = make_double2(0.0, 0.0), zs = zc;
      if (any) {
        zc = make_double2(fv[0] * g[0].x, fv[1] * g[1].x);
        zs = make_double2(s0 * fv[0] * g[0].y, s1 * fv[1] * g[1].y);
        g[0] = cmul(g[0], rho[0]);
        g[1] = cmul(g[1], rho[1]);
      }
      Z[tr * P + m] = zc;
      Z[(tr + nc) * P + m] = zs;
    }
  }
}

// The transposed real-DCT unpack of one packed row at output r (the NDCT's
// big_tr_unpack): za = Z[r mod P], zb = Z[(P - r) mod P], twiddles of kk.
__device__ __forceinline__ double tr_unpack_value(double2 za, double2 zb, double c2, double s2,
                                                  double ch, double sh) {
  const double2 ev = make_double2(0.5 * (za.x + zb.x), 0.5 * (za.y - zb.y));
  const double2 od = make_double2(0.5 * (za.y + zb.y), -0.5 * (za.x - zb.x));
  const double2 V = make_double2(ev.x + od.x * c2 - od.y * s2, ev.y + od.x * s2 + od.y * c2);
  return ch * V.x + sh * V.y;
}

// ---- expansion levels: transposed unpack, out_r += C_r sum_m h_{m,r} (X_cos - X_sin).
// The outputs r in {a, P - a, P + a, 2P - a} read the same two entries a, P - a
// of every packed row: one thread per a in [0, P/2] computes all four.
__global__ void __launch_bounds__(256) asy_tr_unpack_kernel(const __grid_constant__ LevTab lt, int l0,
                                                            int l1, int m0, int nm,
                                                            const double2* __restrict__ Z,
                                                            long long n, size_t nc,
                                                            const double* __restrict__ Cn,
                                                            double* __restrict__ out, size_t ld) {
  const long long P = n / 2;
  const size_t col = blockIdx.y;
  const double nd = (double)n;
  for (long long a = blockIdx.x * (long long)blockDim.x + threadIdx.x; a <= P / 2;
       a += (long long)gridDim.x * blockDim.x) {
    const long long bq = (P - a) & (P - 1);
    const bool four = a != 0 && a != P / 2;
    const int nr = four ? 4 : 2;
    long long r[4];
    bool swp[4];  // the cos rows read (Z[b], Z[a]) instead of (Z[a], Z[b])
    r[0] = a;
    swp[0] = false;
    r[1] = P + a;
    swp[1] = false;
    r[2] = P - a;
    swp[2] = true;
    r[3] = 2 * P - a;
    swp[3] = true;
    double c2[4], s2[4], ch[4], sh[4], h[4], acc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (e >= nr) break;
      sincospi(-2.0 * (double)r[e] / nd, &s2[e], &c2[e]);  // e^{-2 pi i r/N}
      sincospi((double)r[e] / (2.0 * nd), &sh[e], &ch[e]);  // e^{i pi r/(2N)}
      acc[e] = 0.0;
    }
    for (int lv = 0; lv < l1 - l0; ++lv) {
      const long long nu = lt.nu[l0 + lv];
#pragma unroll
      for (int e = 0; e < 4; ++e) h[e] = 1.0;
      for (int tm = 1; tm < m0; ++tm) {
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = h[e] * lt.hk[tm] * __drcp_rn((double)r[e] + (double)tm + 0.5);
      }
      // the four packed entries of term m0 + i, prefetched one term ahead
      auto zrow = [&](int i, double2& ca, double2& cb, double2& sa, double2& sb) {
        const size_t tr = ((size_t)(lv * nm + i) * 2) * nc + col;
        const double2* Zc = Z + tr * P;
        const double2* Zs = Z + (tr + nc) * P;
        ca = __ldcs(Zc + a);
        cb = __ldcs(Zc + bq);
        sa = __ldcs(Zs + a);
        sb = __ldcs(Zs + bq);
      };
      double2 nca, ncb, nsa, nsb;
      zrow(0, nca, ncb, nsa, nsb);
      for (int tm = m0; tm < m0 + nm; ++tm) {
        const double2 ca = nca, cb = ncb, sa = nsa, sb = nsb;
        if (tm + 1 < m0 + nm) zrow(tm + 1 - m0, nca, ncb, nsa, nsb);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (e >= nr) break;
          if (tm > 0) h[e] = h[e] * lt.hk[tm] * __drcp_rn((double)r[e] + (double)tm + 0.5);
          if (r[e] < nu) continue;
          const double xc = swp[e] ? tr_unpack_value(cb, ca, c2[e], s2[e], ch[e], sh[e])
                                   : tr_unpack_value(ca, cb, c2[e], s2[e], ch[e], sh[e]);
          // the sine rows: kk = N - r, e^{-2 pi i kk/N} = conj, e^{i pi kk/(2N)} = i conj
          const double xs = r[e] == 0 ? 0.0
                            : swp[e]  ? tr_unpack_value(sa, sb, c2[e], -s2[e], sh[e], ch[e])
                                      : tr_unpack_value(sb, sa, c2[e], -s2[e], sh[e], ch[e]);
          acc[e] = __fma_rn(h[e], xc - xs, acc[e]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (e >= nr) break;
      if (r[e] < lt.nu[l0]) continue;
      out[col * ld + r[e]] += __ldg(Cn + r[e]) * acc[e];
    }
  }
}

// ---- small elementwise kernels --------------------------------------------
// chat_j = (2 - delta_j0)/N * g_j (the scaled DCT-II of the values, and the
// scaling of the transpose's input)
__global__ void asy_cheb_scale_kernel(const double* __restrict__ in, double* __restrict__ out,
                                      long long n, size_t ld, size_t cols) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n * (long long)cols) return;
  const long long col = i / n, j = i - col * n;
  out[col * ld + j] = in[col * ld + j] * ((j == 0 ? 1.0 : 2.0) / (double)n);
}

}  // namespace

struct L2CAsy {
  size_t n = 0;
  int M = 0;
  LevTab lt{};
  RecTab rt{};
  int nbands = 0;
  RecBand band_all[kMaxBands];  // the bands in term order (stage terms L M ...)
  double* Cn = nullptr;
  double2* ab = nullptr;
  long long rec_steps = 0;  // (point, degree) recurrence steps
  // The chunk start states (P, d) of the recurrence depend on the points and
  // the bands only, not on the data: kept per term range [t_lo, t_hi) after
  // the first call (a rank of the term-parallel C5 always asks for the same
  // range), so later calls skip the transfer-matrix and prefix passes (2^20:
  // 0.62 of 2.78 ms per DLT; 2^26: 20.9 of 188 ms).
  struct Starts {
    int t_lo, t_hi;
    double2* St;
  };
  mutable std::mutex mu;
  mutable std::vector<Starts> starts;
  bool keep_starts = true;
};

namespace {

double log_c(double n) {  // log C_n
  return std::log(4.0 / kPi) + std::lgamma(n + 1.0) + std::lgamma(1.5) - std::lgamma(n + 1.5);
}
double log_h(int m, double n) {
  double s = 0.0;
  for (int j = 1; j <= m; ++j) s += std::log((j - 0.5) * (j - 0.5) / (j * (n + j + 0.5)));
  return s;
}
// smallest sin t at which the M-term remainder for every n >= nu is <= eps
double s_min(double nu, int M, double eps) {
  return 0.5 * std::exp((std::log(2.0) + log_c(nu) + log_h(M, nu) - std::log(eps)) / (M + 0.5));
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

}  // namespace

bool l2c_asy_supported(size_t n) {
  return n >= 1024 && n <= (size_t(1) << 26) && (n & (n - 1)) == 0;
}

L2CAsy* l2c_asy_create(size_t n, const double* s, cudaStream_t st, int M, int R, int max_levels) {
  if (!l2c_asy_supported(n)) return nullptr;
  if (M <= 0) M = env_int("FLB_ASY_M", 10);
  if (R <= 0) R = env_int("FLB_ASY_R", 12);
  if (max_levels < 0) max_levels = env_int("FLB_ASY_LEVELS", kMaxLev);
  M = std::min(std::max(M, 2), kMaxM);
  R = std::max(R, 2);
  const double eps = std::ldexp(1.0, -54);
  const long long N = (long long)n, H = N / 2;
  auto* f = new L2CAsy;
  f->n = n;
  f->M = M;
  // levels (tools/asy_model.py:levels)
  std::vector<long long> nus;
  std::vector<double> S;
  for (long long nu = 8; nu < N && (int)nus.size() < std::min(max_levels, kMaxLev);) {
    const double sm = s_min((double)nu, M, eps);
    if (sm < 1.0) {
      nus.push_back(nu);
      S.push_back(sm);
    }
    nu = nus.empty() ? nu + 8 : nu * R;
  }
  // first pair with sin t_p >= S_l (t_p = (p + 1/2) pi / N increasing)
  auto first_pair = [&](double sl) {
    long long lo = 0, hi = H;
    while (lo < hi) {
      const long long mid = (lo + hi) / 2;
      if (std::sin(kPi * ((double)mid + 0.5) / (double)N) >= sl)
        hi = mid;
      else
        lo = mid + 1;
    }
    return lo;
  };
  LevTab& lt = f->lt;
  lt.M = M;
  lt.pb[0] = H;
  int L = 0;
  for (size_t l = 0; l < nus.size(); ++l) {
    const long long p = first_pair(S[l]);
    if (p >= lt.pb[L]) continue;  // no point left for this level
    lt.nu[L] = nus[l];
    lt.pb[L + 1] = p;
    ++L;
  }
  lt.L = L;
  for (int t = 1; t < M; ++t) lt.hk[t] = (t - 0.5) * (t - 0.5) / t;
  // recurrence bands: [0, pb[L]) to N, then level L-1 ... 0
  RecTab& rt = f->rt;
  rt.nb = 0;
  // chains of up to chain_cap steps run whole, longer ones in chunks of it.
  // A chain is sequential (~36 cycles per step: one 16384-step chain alone is
  // 0.3 ms), and the chunks' start states are kept by the plan, so chunking
  // costs nothing per call: short chunks up to 2^22 (N / 256 in [1024, 8192]:
  // 2^17 0.273 -> 0.251 ms, 2^20 1.62 -> 1.50, 2^22 6.98 -> 6.35 forward),
  // 65536 above (2^24, 2^26: no difference between 8192 and 65536; fewer
  // start-state slots). FLB_ASY_CHAIN overrides.
  long long chain_cap = N < (1ll << 23) ? std::min<long long>(8192, std::max<long long>(1024, N / 256))
                                        : 65536;
  if (env_int("FLB_ASY_CHAIN", 0) > 0) chain_cap = (env_int("FLB_ASY_CHAIN", 0) + 31) / 32 * 32;
  long long wb = 0, xb = 0, ib = 0, gb = 0, rb = 0;
  auto add_band = [&](long long p0, long long p1, long long nu) {
    if (p1 <= p0) return;
    RecBand& B = rt.b[rt.nb++];
    B.p0 = p0;
    B.p1 = p1;
    B.nu = nu;
    // chains up to `cap` degrees run whole (no transfer matrices); longer
    // ones in chunks of `cap`
    const long long lc = nu <= chain_cap ? (nu + 31) / 32 * 32 : chain_cap;
    B.lc = (int)lc;
    B.Q = (int)((nu + lc - 1) / lc);
    B.G = (int)((p1 - p0 + kPairsPerWarp - 1) / kPairsPerWarp);
    // transposed workers per chunk: ~1024 warps per band, partial rows <= 2^25 entries
    const long long g2 = (B.G + kTrGroups - 1) / kTrGroups;
    long long W = std::min<long long>(g2, std::max<long long>(1, (1024 + B.Q - 1) / B.Q));
    while (W > 1 && (long long)B.Q * W * lc > (1ll << 25)) W = (W + 1) / 2;
    B.W = (int)W;
    B.wbase = wb;
    B.xbase = xb;
    B.ibase = ib;
    B.gbase = gb;
    B.rbase = rb;
    wb += (long long)B.G * B.Q;
    xb += (long long)B.Q * B.W;
    ib += (long long)B.G * B.Q * kPairsPerWarp;
    gb += (long long)B.G * kPairsPerWarp;
    rb += (long long)B.Q * B.W * lc;
    f->rec_steps += 2 * (p1 - p0) * nu;
  };
  add_band(0, lt.pb[L], N);
  for (int l = L - 1; l >= 0; --l) add_band(lt.pb[l + 1], lt.pb[l], lt.nu[l]);
  rt.nwarps = wb;
  rt.nxwarps = xb;
  rt.nslots = ib;
  rt.ngslots = gb;
  rt.nrows = rb;
  f->nbands = rt.nb;
  for (int b = 0; b < rt.nb; ++b) f->band_all[b] = rt.b[b];
  FLB_CUDA(cudaMalloc(&f->Cn, n * sizeof(double)));
  FLB_CUDA(cudaMalloc(&f->ab, n * sizeof(double2)));
  asy_tables_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(N, s, f->Cn, f->ab);
  note_launch("asy_tables_kernel");
  return f;
}

void l2c_asy_destroy(L2CAsy* f) {
  if (!f) return;
  if (f->Cn) cudaFree(f->Cn);
  if (f->ab) cudaFree(f->ab);
  for (const L2CAsy::Starts& c : f->starts) cudaFree(c.St);
  delete f;
}

void l2c_asy_one_shot(L2CAsy* f) {
  if (f) f->keep_starts = false;
}

L2CAsyInfo l2c_asy_info(const L2CAsy& f) {
  return {f.M, f.lt.L, 2 * f.M * f.lt.L, (double)f.rec_steps / (double)f.n};
}

namespace {

template <class T>
struct AsyncBuf {
  T* p = nullptr;
  cudaStream_t s;
  AsyncBuf(size_t count, cudaStream_t st) : s(st) {
    if (count) FLB_CUDA(cudaMallocAsync(&p, count * sizeof(T), st));
  }
  ~AsyncBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  AsyncBuf(const AsyncBuf&) = delete;
  AsyncBuf& operator=(const AsyncBuf&) = delete;
};

unsigned grid_for(long long work, int threads, long long cap = 1 << 20) {
  return (unsigned)std::max<long long>(1, std::min<long long>((work + threads - 1) / threads, cap));
}

// levels per batch of the expansion's transforms (Z + FFT scratch within a
// fixed 12 GiB budget: the same batching, hence the same scratch sizes, on
// every call)
int levels_per_batch(const L2CAsy& f, size_t nc) {
  const size_t per_level = (size_t)2 * f.M * nc * (f.n / 2) * sizeof(double2) * 2;
  const size_t budget = size_t(12) << 30;
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)std::max(f.lt.L, 1), budget / per_level));
}

// Grow the stream-ordered pool to a call's whole scratch in one allocation
// (freed at once, kept by the pool's release threshold): the call's buffers
// are then carved from memory the pool already holds, instead of an
// occasional mid-call pool growth (a ~9 ms outlier at 2^20).
void reserve_scratch(size_t bytes, cudaStream_t s) {
  void* p = nullptr;
  if (bytes && cudaMallocAsync(&p, bytes, s) == cudaSuccess) cudaFreeAsync(p, s);
  cudaGetLastError();
}

// The recurrence's scratch (allocated on the caller's stream before the fork).
struct RecBufs {
  double4* T;   // chunk transfer matrices
  double2* St;  // chunk start states
  double2* Ep;  // forward: per (pair, chunk) even / odd partial sums
  double* R;    // transposed: per-worker partial rows
};

// The recurrence runs on an auxiliary stream beside the expansion's level
// transforms: it is FP64-issue-bound, they are HBM-bound.
cudaStream_t aux_stream() {
  static std::mutex mu;
  static std::map<int, cudaStream_t> per_dev;
  int dev = 0;
  FLB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    // the lowest priority: the levels' kernels (the caller's stream) take
    // the SMs first, the recurrence's CTAs fill what they leave
    int least = 0, greatest = 0;
    FLB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    cudaStream_t st;
    FLB_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, least));
    it = per_dev.emplace(dev, st).first;
  }
  return it->second;
}

// The chunk start states of the bands in rt (data-independent): per chunk a
// 2x2 transfer matrix, then the sequential prefix over each pair's chunks.
void recurrence_starts(const L2CAsy& f, const RecTab& rt, double4* T, double2* St, cudaStream_t s) {
  if (rt.nb == 0) return;
  const double nd = (double)f.n;
  asy_rec_transfer_kernel<<<grid_for(rt.nwarps * 32, kRecThreads, 1ll << 31), kRecThreads, 0, s>>>(
      rt, f.ab, nd, T);
  note_launch("asy_rec_transfer_kernel");
  asy_rec_prefix_kernel<<<grid_for(rt.ngslots, 128, 1ll << 31), 128, 0, s>>>(rt, T, St, nd);
  note_launch("asy_rec_prefix_kernel");
}

void recurrence_chains(const L2CAsy& f, const RecTab& rt, int transpose, const double* x, size_t ld,
                       size_t cols, const RecBufs& b, cudaStream_t s) {
  if (rt.nb == 0) return;
  const long long n = (long long)f.n;
  const double nd = (double)n;
  if (!transpose) {
    asy_rec_fwd_kernel<<<dim3(grid_for(rt.nwarps * 32, kRecThreads, 1ll << 31), (unsigned)cols),
                         kRecThreads, 0, s>>>(rt, f.ab, x, ld, b.St, b.Ep, nd);
    note_launch("asy_rec_fwd_kernel");
  } else {
    asy_rec_tr_kernel<<<dim3(grid_for(rt.nxwarps * 32, kRecThreads, 1ll << 31), (unsigned)cols),
                        kRecThreads, 0, s>>>(rt, f.ab, x, ld, b.St, b.R, nd, n);
    note_launch("asy_rec_tr_kernel");
  }
}

// forward: F (zeroed, the levels added) += the recurrence's sums
void recurrence_forward_finish(const L2CAsy& f, const RecTab& rt, const RecBufs& b, double* F, size_t ld,
                               size_t cols, cudaStream_t s) {
  if (rt.nb == 0) return;
  asy_rec_fwd_finish_kernel<<<dim3(grid_for(rt.ngslots, 256, 1ll << 31), (unsigned)cols), 256, 0, s>>>(
      rt, b.Ep, F, ld, (long long)f.n);
  note_launch("asy_rec_fwd_finish_kernel");
}

// transposed: out (the levels added) += the recurrence's rows, then (n + 1/2)
// (also without bands: the scaling of the whole output)
void recurrence_transpose_finish(const L2CAsy& f, const RecTab& rt, const RecBufs& b, double* out,
                                 size_t ld, size_t cols, int scale_half, cudaStream_t s) {
  const long long n = (long long)f.n;
  asy_rec_tr_finish_kernel<<<dim3((unsigned)(n / 32), (unsigned)cols), 256, 0, s>>>(rt, b.R, out, ld, n,
                                                                                   scale_half);
  note_launch("asy_rec_tr_finish_kernel");
}

// Event fork / join between the caller's stream and the recurrence stream.
struct Fork {
  cudaStream_t main, aux;
  cudaEvent_t ev[2];
  Fork(cudaStream_t s) : main(s), aux(aux_stream()) {
    for (cudaEvent_t& e : ev) FLB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    FLB_CUDA(cudaEventRecord(ev[0], main));
    FLB_CUDA(cudaStreamWaitEvent(aux, ev[0], 0));
  }
  void join() {
    FLB_CUDA(cudaEventRecord(ev[1], aux));
    FLB_CUDA(cudaStreamWaitEvent(main, ev[1], 0));
  }
  ~Fork() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

}  // namespace

int l2c_asy_terms(const L2CAsy& f) { return f.lt.L * f.M + f.nbands; }

double l2c_asy_term_cost(const L2CAsy& f, int term) {
  // measured on one B200 at 2^26: a level term (two length-N transforms with
  // their pack / unpack) ~27.7 ps per coefficient, a recurrence pair-step ~0.67 ps
  if (term < f.lt.L * f.M) return 27.7 * (double)f.n;
  const RecBand& B = f.band_all[term - f.lt.L * f.M];
  return 0.67 * (double)(B.p1 - B.p0) * (double)B.nu;
}

void l2c_asy_apply(const L2CAsy& f, int transpose, const double* in, double* out, size_t cols,
                   size_t ld, int scale_half, cudaStream_t s, int t_lo, int t_hi) {
  if (cols == 0) return;
  const long long n = (long long)f.n, P = n / 2;
  const int log2n = __builtin_ctzll((unsigned long long)n);
  const int L = f.lt.L, M = f.M, LM = L * M;
  if (t_hi < 0) t_hi = l2c_asy_terms(f);
  const bool full = t_lo <= 0 && t_hi >= l2c_asy_terms(f);
  // the level segments (level, first term, terms) of this call: whole levels
  // batched when all terms run, else one level at a time
  struct Seg {
    int l0, l1, m0, nm;
  };
  std::vector<Seg> segs;
  const int lpb = levels_per_batch(f, cols);
  if (full) {
    for (int l0 = 0; l0 < L; l0 += lpb) segs.push_back({l0, std::min(L, l0 + lpb), 0, M});
  } else {
    for (int l = 0; l < L; ++l) {
      const int a = std::max(t_lo, l * M), b = std::min(t_hi, (l + 1) * M);
      if (a < b) segs.push_back({l, l + 1, a - l * M, b - a});
    }
  }
  // the recurrence bands of this call
  RecTab rt{};
  if (full) {
    rt = f.rt;
  } else {
    long long wb = 0, xb = 0, ib = 0, gb = 0, rb = 0;
    for (int bi = 0; bi < f.nbands; ++bi) {
      const int term = LM + bi;
      if (term < t_lo || term >= t_hi) continue;
      RecBand B = f.band_all[bi];
      B.wbase = wb;
      B.xbase = xb;
      B.ibase = ib;
      B.gbase = gb;
      B.rbase = rb;
      wb += (long long)B.G * B.Q;
      xb += (long long)B.Q * B.W;
      ib += (long long)B.G * B.Q * kPairsPerWarp;
      gb += (long long)B.G * kPairsPerWarp;
      rb += (long long)B.Q * B.W * B.lc;
      rt.b[rt.nb++] = B;
    }
    rt.nwarps = wb;
    rt.nxwarps = xb;
    rt.nslots = ib;
    rt.ngslots = gb;
    rt.nrows = rb;
  }
  size_t zlev = 0;
  for (const Seg& g : segs) zlev = std::max(zlev, (size_t)(g.l1 - g.l0) * g.nm);
  const size_t per_term = (size_t)2 * cols * P;
  reserve_scratch(2 * zlev * per_term * sizeof(double2) + 2 * ld * cols * sizeof(double) +
                      (size_t)rt.nslots * (sizeof(double4) + sizeof(double2) * (1 + cols)) +
                      (size_t)rt.nrows * cols * sizeof(double) + (size_t(64) << 20),
                  s);
  AsyncBuf<double2> Z(zlev * per_term, s);
  AsyncBuf<double2> S(zlev * per_term, s);
  AsyncBuf<double> F(ld * cols, s);
  // the start states: from the plan's cache, or computed now (and kept, up to
  // kMaxStarts term ranges per plan; the first call of a range synchronises
  // once before publishing them to other threads / streams)
  constexpr size_t kMaxStarts = 4;
  double2* st_cached = nullptr;
  bool st_keep = false;
  if (rt.nslots > 0 && f.keep_starts) {
    const int k_lo = full ? 0 : t_lo, k_hi = full ? l2c_asy_terms(f) : t_hi;
    std::lock_guard<std::mutex> lock(f.mu);
    for (const L2CAsy::Starts& c : f.starts)
      if (c.t_lo == k_lo && c.t_hi == k_hi) st_cached = c.St;
    if (!st_cached && f.starts.size() < kMaxStarts) {
      double2* p = nullptr;
      if (cudaMalloc(&p, (size_t)rt.nslots * sizeof(double2)) == cudaSuccess) {
        AsyncBuf<double4> T0(rt.nslots, s);
        recurrence_starts(f, rt, T0.p, p, s);
        FLB_CUDA(cudaStreamSynchronize(s));
        f.starts.push_back({k_lo, k_hi, p});
        st_cached = p;
      } else {
        cudaGetLastError();
      }
    }
    st_keep = st_cached != nullptr;
  }
  AsyncBuf<double4> T(st_keep ? 0 : rt.nslots, s);
  AsyncBuf<double2> St(st_keep ? 0 : rt.nslots, s);
  if (!st_keep) recurrence_starts(f, rt, T.p, St.p, s);
  AsyncBuf<double2> Ep(transpose ? 0 : rt.nslots * cols, s);
  AsyncBuf<double> R(transpose ? rt.nrows * cols : 0, s);
  const RecBufs rb{T.p, st_keep ? st_cached : St.p, Ep.p, R.p};
  const unsigned gp = grid_for(P, 256, 4096);
  if (!transpose) {
    // values at the cheb1 points: the recurrence's sums, then the levels'
    // (on one stream: beside the levels' transforms the forward chains ran
    // slower -- 2^20 2.9 vs 2.2 ms, 2^22 11.9 vs 10.5 ms)
    FLB_CUDA(cudaMemset2DAsync(F.p, ld * sizeof(double), 0, n * sizeof(double), cols, s));
    recurrence_chains(f, rt, 0, in, ld, cols, rb, s);
    recurrence_forward_finish(f, rt, rb, F.p, ld, cols, s);
    for (const Seg& g : segs) {
      asy_fwd_pack_kernel<<<dim3(gp, (unsigned)cols, (unsigned)(g.l1 - g.l0)), 256, 0, s>>>(
          f.lt, g.l0, g.m0, g.nm, in, ld, f.Cn, n, cols, Z.p);
      note_launch("asy_fwd_pack_kernel");
      fft_pow2(Z.p, S.p, log2n - 1, (size_t)2 * g.nm * cols * (g.l1 - g.l0), true, s);
      const long long pts = 2 * (f.lt.pb[g.l0] - f.lt.pb[g.l1]);
      asy_fwd_unpack_kernel<<<dim3(grid_for(pts, 256, 8192), (unsigned)cols), 256, 0, s>>>(
          f.lt, g.l0, g.l1, g.m0, g.nm, Z.p, n, cols, F.p, ld);
      note_launch("asy_fwd_unpack_kernel");
    }
    // chat = (2 - delta_j0)/N sum_k f_k cos(j t_k): dct_iii_transpose + scaling
    fast_trig(FL_DCT_III_T, f.n, F.p, out, cols, ld, s);
    asy_cheb_scale_kernel<<<grid_for(n * (long long)cols, 256, 1ll << 31), 256, 0, s>>>(out, out, n, ld,
                                                                                         cols);
    note_launch("asy_cheb_scale_kernel");
  } else {
    // M^T = E^T D^T: values f = dct_iii((2 - delta_j0)/N g), then the transposed evaluation
    AsyncBuf<double> G(ld * cols, s);
    asy_cheb_scale_kernel<<<grid_for(n * (long long)cols, 256, 1ll << 31), 256, 0, s>>>(in, G.p, n, ld,
                                                                                         cols);
    note_launch("asy_cheb_scale_kernel");
    fast_trig(FL_DCT_III, f.n, G.p, F.p, cols, ld, s);
    FLB_CUDA(cudaMemset2DAsync(out, ld * sizeof(double), 0, n * sizeof(double), cols, s));
    // the transposed recurrence on the auxiliary stream beside the levels
    // (2^20 2.6 -> 2.2 ms, 2^22 11.5 -> 9.4, 2^24 52.9 -> 44.1; 2^26 unchanged)
    Fork fk(s);
    recurrence_chains(f, rt, 1, F.p, ld, cols, rb, fk.aux);
    for (const Seg& g : segs) {
      asy_tr_pack_kernel<<<dim3(gp, (unsigned)cols, (unsigned)(g.l1 - g.l0)), 256, 0, s>>>(
          f.lt, g.l0, g.m0, g.nm, F.p, ld, n, cols, Z.p);
      note_launch("asy_tr_pack_kernel");
      fft_pow2(Z.p, S.p, log2n - 1, (size_t)2 * g.nm * cols * (g.l1 - g.l0), false, s);
      asy_tr_unpack_kernel<<<dim3(grid_for(P / 2 + 1, 256, 8192), (unsigned)cols), 256, 0, s>>>(
          f.lt, g.l0, g.l1, g.m0, g.nm, Z.p, n, cols, f.Cn, out, ld);
      note_launch("asy_tr_unpack_kernel");
    }
    fk.join();
    recurrence_transpose_finish(f, rt, rb, out, ld, cols, scale_half, s);
  }
}

}  // namespace flb
