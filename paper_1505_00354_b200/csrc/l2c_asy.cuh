// Asymptotic-expansion Legendre <-> Chebyshev conversion for large N
// (Hale & Townsend 2014, the fast leg2cheb the paper cites; north-star
// subsystem 2). Replaces the O(N^2) loops of conversion.hpp:100-140 for
// single vectors / few columns at power-of-two N.
//
// chat = M c is computed as the Chebyshev coefficients of the Legendre
// series sampled at the N cheb1 points t_k = (k + 1/2) pi / N:
//   f_k = sum_n c_n P_n(cos t_k),   chat_j = (2 - delta_j0)/N sum_k f_k cos(j t_k).
// P_n(cos t) = C_n sum_{m<M} h_{m,n} cos((n+m+1/2) t - (m+1/2) pi/2) / (2 sin t)^{m+1/2} + R_M
// for the degrees n >= nu_l of the point's level l (|R_M| <= eps there), so each
// of the M terms is a DCT-III and a DST-III of the diagonally scaled input
// (c_n C_n h_{m,n}, n >= nu_l) with a diagonal output weight; the degrees below
// a point's cutoff come from the three-term recurrence (a chunked, transfer-
// matrix-parallel warp kernel). M^T is the exact transpose of the same steps.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace flb {

struct L2CAsy;

// n: a power of two in [2^10, 2^26]; s: the device scaled Lambda table
// (s_j = Lambda(j)/Lambda(0), n entries). M (expansion terms), R (level
// ratio), max_levels (-1: all levels the tolerance allows; fewer trade
// length-N transforms for recurrence steps): 0 / -1 = defaults
// (FLB_ASY_M / FLB_ASY_R / FLB_ASY_LEVELS override them).
L2CAsy* l2c_asy_create(size_t n, const double* s, cudaStream_t st, int M = 0, int R = 0,
                       int max_levels = -1);
void l2c_asy_destroy(L2CAsy* f);
bool l2c_asy_supported(size_t n);
// Size from which the plan's FAST conversion mode uses the expansion instead of
// Toeplitz-Hankel (single vectors / <= 16 columns): with the chunk start
// states kept by the plan (and its recurrence in short chunks) it wins from
// 2^16 (0.148 vs 0.189 ms; 2^17 0.25 vs 0.32; 2^19 0.68 vs 1.30; 2^15 ties
// at 0.12, 2^14 Toeplitz-Hankel wins 0.097 vs 0.115). The free function
// (a new table per call, nothing kept) switches at kL2CAsyMinFree.
constexpr size_t kL2CAsyMin = size_t(1) << 16;
constexpr size_t kL2CAsyMinFree = size_t(1) << 20;
// A per-call object (fl_leg2cheb): do not keep the start states.
void l2c_asy_one_shot(L2CAsy* f);

// out = M in (transpose 0) or M^T in (1, optional (n + 1/2) output scaling);
// columns of stride ld; in and out must not alias.
// t_lo / t_hi: only the terms [t_lo, t_hi) (a partial sum; the term-parallel
// multi-GPU DLT splits them over ranks): terms [0, L M) are the expansion's
// (level l = t / M, m = t % M) DCT/DST pairs, the next ones the recurrence's
// bands of points (l2c_asy_terms in all, l2c_asy_term_cost their relative cost).
void l2c_asy_apply(const L2CAsy& f, int transpose, const double* in, double* out, size_t cols,
                   size_t ld, int scale_half, cudaStream_t st, int t_lo = 0, int t_hi = -1);
int l2c_asy_terms(const L2CAsy& f);
double l2c_asy_term_cost(const L2CAsy& f, int term);

struct L2CAsyInfo {
  int M, levels, transforms;   // transforms: length-N real DCT/DST per column
  double rec_steps_per_n;      // recurrence (point, degree) steps / N
};
L2CAsyInfo l2c_asy_info(const L2CAsy& f);

}  // namespace flb
