// Distributed four-step NDCT (BASELINE config C5 sharded over P ranks, one
// process per GPU): the Chebyshev-expansion NDCT of one vector of
// length N (power of two) whose input and output are spread over P ranks,
// each term's N/2-point complex FFT a four-step over the ranks with ONE
// all-to-all per group of terms (the caller's NCCL collective) in between.
//
//   L = N/2 = L1 L2,  m = m1 + L1 m2 (packed input),  p = k2 + L2 k1 (output)
//   z[k2 + L2 k1] = sum_{m1} e^{2 pi i m1 k1/L1} e^{2 pi i m1 k2/L} sum_{m2} Z[m1 + L1 m2] e^{2 pi i m2 k2/L2}
//
// Rank r owns (a) on the coefficient side the residues m1 of a symmetric set
// S_r = {j, L1 - j : j in [r h, (r+1) h)} (+ L1/2 on the last rank), h =
// L1/(2P): the Makhoul pack of entry m reads c at m, N - m, m + L, L - m,
// whose residues mod L1 are +-m1, so the pack and the transposed unpack are
// local; (b) on the value side the k2 block [r KB, (r+1) KB), KB = L2/P, with
// every k1. Layouts (rank-local):
//   residue layout   chat[i][j] = c_{res_i + L1 j}, j < 2 L2
//   exchange (coef)  [peer][t][i_src][k2 - peer... ] complex, see dist_ndct in fast_ndct.cu
//   exchange (value) [peer][g][u][k2l][b] doubles, B/P per peer (uniform)
// The value side's natural blocks (rank d: k in [d B, (d+1) B), B = N/P) map
// to two contiguous p ranges per block, so the final all-to-all is uniform.
// Requirements: P a power of two, 2P <= L1, L1, L2 <= 8192 (N <= 2^27).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "fast_ndct.cuh"

namespace flb {

struct FsLayout;

struct FsInfo {
  size_t n, L, L1, L2, KB, B;
  size_t nres;            // residues of this rank
  size_t res_max;         // max residues over ranks
  int world, rank;
};

FsLayout* fs_create(size_t n, int world, int rank);  // throws Error on unsupported shapes
void fs_destroy(FsLayout* f);
FsInfo fs_info(const FsLayout& f);
// complex elements this rank sends to / receives from `peer` per term in the
// coefficient-side exchange (forward: send nres_me KB, recv nres_peer KB;
// transpose: the other way round)
size_t fs_coef_count(const FsLayout& f, int transpose, int peer, int send);

// natural full vector -> [dest][res_max * 2 L2] (zero padded) for the
// reduce-scatter into residue layouts, and back (all-gathered -> natural)
void fs_to_residue(const FsLayout& f, const double* full, double* send, cudaStream_t s);
void fs_from_residue(const FsLayout& f, const double* gathered, double* full, cudaStream_t s);

// forward NDCT, terms [t0, t1): part 1 (pack, L2-point FFTs, twiddle, into the
// exchange buffer), part 2 (exchange buffer -> L1-point FFTs -> weighted unpack
// accumulated into the value-side exchange layout `fx`; first: store)
void fs_fwd1(const FsLayout& f, const FastNdct& p, int t0, int t1, const double* chat,
             double2* send, double2* work, int* nonfinite, cudaStream_t s);
void fs_fwd2(const FsLayout& f, const FastNdct& p, int t0, int t1, const double2* recv,
             double2* work, double* fx, int first, cudaStream_t s);
// value side: exchange layout <-> this rank's natural block
void fs_values_from_exchange(const FsLayout& f, const double* fx, double* block, cudaStream_t s);
void fs_values_to_exchange(const FsLayout& f, const double* block, double* fx, cudaStream_t s);
// transposed NDCT of mult . g: part 1 (weighted pack from the value-side
// exchange layout, L1-point FFTs, twiddle, into the exchange buffer), part 2
// (L2-point FFTs, transposed unpack accumulated into the residue layout)
void fs_tr1(const FsLayout& f, const FastNdct& p, const double* mult, int t0, int t1,
            const double* gx, double2* send, double2* work, int* nonfinite, cudaStream_t s);
void fs_tr2(const FsLayout& f, const FastNdct& p, int t0, int t1, const double2* recv,
            double2* work, double* chat, int first, cudaStream_t s);

}  // namespace flb
