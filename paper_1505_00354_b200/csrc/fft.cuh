// Batched power-of-two complex fp64 FFT engine (the replacement of FFTW's
// codelets behind trig.hpp:31-47). Used by the generic chirp-z DCT/DST path
// (any N, both grid kinds). Forward = e^{-2 pi i jk/P}, inverse = e^{+...},
// both unnormalised.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "common.cuh"

namespace flb {

// Device table e^{-2 pi i m / P}, m < P (cached per device and P).
const double2* twiddle_table(int log2p);

// In-place batched FFT of `batch` contiguous rows of length 2^log2p.
// `scratch` must hold batch * 2^log2p elements when log2p > 13 (six-step).
void fft_pow2(double2* data, double2* scratch, int log2p, size_t batch, bool inverse,
              cudaStream_t s);

constexpr int kMaxSmemLog2 = 13;  // 8192 points = 128 KiB of double2 per CTA
constexpr int kMaxLog2 = 26;

// The multi-pass NDCT's forward transforms with the unpack fused into the last
// (row) pass (fast_ndct.cu, N > 16384): `data` holds nt * nc packed rows of
// 2^log2p points (row tz * nc + col); all passes but the last run as in
// fft_pow2, then one CTA per group of adjacent lines and column runs the row
// pass of every term in turn and accumulates
//   out[col][kx(m)] (+)= sum_tz wp[tz][m].x Re X_tz[m],  out[col][ky(m)] likewise with Im,
// kx, ky = 4m, 4m + 2 (m < P/2) or 2N - 4m - 1, 2N - 4m - 3 (the real-DCT
// packing's output order, N = 2P), in registers: the transformed rows are
// never written (one write and one read of all terms x columns less).
struct NdctUnpack {
  const double2* wp;  // [nt][P] output weights (signs folded in)
  double* out;        // columns of stride ld
  size_t ld, nc;
  int nt, first;      // first: store, else add to out
};
// The transposed direction's counterpart: the pack fused into the first pass's
// loads. Row tz * nc + col of the transform is wp[tz][m] (.) G[col][m]
// (componentwise: real part with real part), G the column's weighted input in
// packed-entry order; the packed rows are never written or read.
struct NdctTrPack {
  const double2* wp;  // [nt][P]
  const double2* G;   // [nc][P]
  size_t nc;
  int nt;
};
void fft_pow2_ndct_tr_pack(double2* data, double2* scratch, int log2p, bool inverse,
                           const NdctTrPack& a, cudaStream_t s);
bool fft_pow2_ndct_unpack_ok(int log2p);
void fft_pow2_ndct_unpack(double2* data, double2* scratch, int log2p, bool inverse,
                          const NdctUnpack& a, cudaStream_t s);

// ---- fused Toeplitz-Hankel sweep (l2c_fast.cu) for 2^log2p > 8192 -------------
// One batched sweep over rank pairs q < pairs computes, per pair,
//   W_q = IFFT(FFT(V_q) . S~),  V_q[b] = (l_{ra}(b) u_b, l_{ra+1}(b) u_b) (b < np, else 0),
// ra = ra0 + 2q, u_b = x[2b+p] (doubled for the transpose when 2b+p != 0),
// S~ = conj(S) (forward) or S (transpose), into V (natural order,
// unnormalised). The packing is done by the first FFT pass's loads, and the
// last forward pass, the symbol product and the first inverse pass are one
// row pass (the spectrum never leaves shared memory in transposed order):
// 2 + 2 (P <= 2^24) or 3 + 2 sweeps instead of pack + 2 + mul + 2 + ... .
// (Folding the l_r accumulation into the last inverse pass was measured
// slower: its register footprint halves the resident CTAs.)
struct ThArgs {
  const double* x;
  int p;
  unsigned long long np;
  const double* ell;
  int K, ra0, transpose;
  const double2* sym;   // the symbol spectrum in th_symbol_layout order
};
// Reorder a natural-order spectrum (length 2^log2p) for the fused sweep's row
// pass (scratch: 2^log2p elements).
void th_symbol_layout(double2* sym, double2* scratch, int log2p, cudaStream_t s);
// V, S: pairs * 2^log2p elements each; W is left in V.
void th_sweep(const ThArgs& a, int log2p, size_t pairs, double2* V, double2* S, cudaStream_t s);

// Register-resident small DFTs (natural order in and out).
template <bool INV>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  const double2 t = a;
  a = make_double2(t.x + b.x, t.y + b.y);
  b = make_double2(t.x - b.x, t.y - b.y);
}

template <bool INV>
__device__ __forceinline__ double2 rot_mi(double2 v) {  // v * (-i) forward, v * (+i) inverse
  return INV ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
  const double2 t0 = make_double2(v0.x + v2.x, v0.y + v2.y);
  const double2 t1 = make_double2(v0.x - v2.x, v0.y - v2.y);
  const double2 t2 = make_double2(v1.x + v3.x, v1.y + v3.y);
  const double2 t3 = rot_mi<INV>(make_double2(v1.x - v3.x, v1.y - v3.y));
  v0 = make_double2(t0.x + t2.x, t0.y + t2.y);
  v2 = make_double2(t0.x - t2.x, t0.y - t2.y);
  v1 = make_double2(t1.x + t3.x, t1.y + t3.y);
  v3 = make_double2(t1.x - t3.x, t1.y - t3.y);
}

template <bool INV>
__device__ __forceinline__ void dft8(double2* v) {
  constexpr double h = 0.70710678118654752440084436210484903928;
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  // w^k, w = e^{-+ 2 pi i / 8}
  const double2 w1o = INV ? make_double2(h * (o1.x - o1.y), h * (o1.x + o1.y))
                          : make_double2(h * (o1.x + o1.y), h * (o1.y - o1.x));
  const double2 w2o = rot_mi<INV>(o2);
  const double2 w3o = INV ? make_double2(-h * (o3.x + o3.y), h * (o3.x - o3.y))
                          : make_double2(h * (o3.y - o3.x), -h * (o3.x + o3.y));
  v[0] = make_double2(e0.x + o0.x, e0.y + o0.y);
  v[4] = make_double2(e0.x - o0.x, e0.y - o0.y);
  v[1] = make_double2(e1.x + w1o.x, e1.y + w1o.y);
  v[5] = make_double2(e1.x - w1o.x, e1.y - w1o.y);
  v[2] = make_double2(e2.x + w2o.x, e2.y + w2o.y);
  v[6] = make_double2(e2.x - w2o.x, e2.y - w2o.y);
  v[3] = make_double2(e3.x + w3o.x, e3.y + w3o.y);
  v[7] = make_double2(e3.x - w3o.x, e3.y - w3o.y);
}

template <int R, bool INV>
__device__ __forceinline__ void dft_r(double2* v) {
  if constexpr (R == 2) {
    dft2<INV>(v[0], v[1]);
  } else if constexpr (R == 4) {
    dft4<INV>(v[0], v[1], v[2], v[3]);
  } else {
    dft8<INV>(v);
  }
}

// Shared-memory rows are padded with one element after every 8 so that the
// stride-8 accesses of the first radix-8 pass are bank-conflict free
// (8 lanes x 16 B fill one 128 B wavefront).
__host__ __device__ constexpr int smem_pad(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int smem_row(int p) { return p + p / 8; }

// One Stockham pass (compile-time Ns and radix R) over a padded
// shared-memory row of P points held by TR = P/E threads, each doing E/R
// radix-R butterflies:
//   v_r = x[j + r P/R] * w_{Ns R}^{r (j mod Ns)};  DFT_R;
//   y[(j/Ns) Ns R + (j mod Ns) + r Ns] = V_r.
//
// Twiddles come from a pass-major table (global, L1/L2-resident): for each pass with
// Ns > 1, entries (r-1) Ns + k hold w_{Ns R}^{r k}, r = 1..R-1, k < Ns, so a
// warp reads consecutive k (bank-conflict free) and the table is only
// sum_passes (R-1) Ns ~ P entries.
// Barrier over the threads that own one row: the whole CTA (GT = 0), one
// warp (GT = 32), or a named barrier `bar` of GT threads (several rows per CTA
// progress independently).
template <int GT>
__device__ __forceinline__ void group_sync(int bar) {
  if constexpr (GT == 0) {
    __syncthreads();
  } else if constexpr (GT == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(GT) : "memory");
  }
}

// The three stages of a pass, usable separately so that a kernel can feed the
// first pass from registers and consume the last pass in registers.
// Input of butterfly q of thread tid: v[q R + r] = x[j + r P/R], j = tid + q TR.
// MIR (two butterflies per thread): j = tid and P/R - 1 - tid instead, so
// that in the last pass (NS = P/R, outputs j + r NS) a thread holds outputs
// m and P - 1 - m together.
template <int P, int E, int R, bool MIR = false>
__device__ __forceinline__ int butterfly_j(int tid, int q) {
  static_assert(!MIR || E / R == 2, "mirrored butterflies: two per thread");
  return MIR ? (q == 0 ? tid : P / R - 1 - tid) : tid + q * (P / E);
}

template <int P, int E, int R, bool MIR = false>
__device__ __forceinline__ void pass_load(double2* v, const double2* s, int tid) {
  constexpr int NB = E / R;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int j = butterfly_j<P, E, R, MIR>(tid, q);
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = s[smem_pad(j + r * (P / R))];
  }
}

// TWP (twiddle powers): instead of loading all R-1 twiddles w^{r k} of a
// butterfly, load w^k (and w^{4k} for R = 8) and form the rest by complex
// products (at most three roundings deep): 2 loads instead of 7 for radix 8,
// 1 instead of 3 for radix 4 -- shared-memory wavefronts traded for FP64 work.
// Only for NS >= 64: below that a warp's twiddle loads hit few distinct
// entries (broadcast, ~1 wavefront) and the products cost more than they save.
template <int P, int E, int R, int NS, bool INV, bool TWP = false, bool MIR = false>
__device__ __forceinline__ void pass_compute(double2* v, int tid, const double2* tw) {
  constexpr int NB = E / R;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int j = butterfly_j<P, E, R, MIR>(tid, q);
    const int k = j & (NS - 1);
    if constexpr (NS > 1 && TWP && NS >= 64 && (R == 8 || R == 4)) {
      double2 w[R];
      w[1] = tw[k];
      if (INV) w[1].y = -w[1].y;
      w[2] = cmul(w[1], w[1]);
      w[3] = cmul(w[2], w[1]);
      if constexpr (R == 8) {
        w[4] = tw[3 * NS + k];
        if (INV) w[4].y = -w[4].y;
        w[5] = cmul(w[4], w[1]);
        w[6] = cmul(w[4], w[2]);
        w[7] = cmul(w[4], w[3]);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) v[q * R + r] = cmul(v[q * R + r], w[r]);
    } else if (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 w = tw[(r - 1) * NS + k];
        if (INV) w.y = -w.y;
        const double2 a = v[q * R + r];
        v[q * R + r] = make_double2(a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x);
      }
    }
    dft_r<R, INV>(&v[q * R]);
  }
}

// Output r of butterfly q goes to index (j - k) R + k + r Ns, k = j mod Ns.
template <int P, int E, int R, int NS>
__host__ __device__ constexpr int pass_out_index(int tid, int q, int r) {
  return ((tid + q * (P / E)) - ((tid + q * (P / E)) & (NS - 1))) * R +
         ((tid + q * (P / E)) & (NS - 1)) + r * NS;
}

template <int P, int E, int R, int NS>
__device__ __forceinline__ void pass_store(const double2* v, double2* s, int tid) {
  constexpr int NB = E / R;
#pragma unroll
  for (int q = 0; q < NB; ++q)
#pragma unroll
    for (int r = 0; r < R; ++r) s[smem_pad(pass_out_index<P, E, R, NS>(tid, q, r))] = v[q * R + r];
}

template <int P, int E, int R, int NS, bool INV, int GT, bool TWP = false>
__device__ __forceinline__ void stockham_pass(double2* s, int tid, const double2* tw, int bar) {
  double2 v[E];
  pass_load<P, E, R>(v, s, tid);
  group_sync<GT>(bar);
  pass_compute<P, E, R, NS, INV, TWP>(v, tid, tw);
  pass_store<P, E, R, NS>(v, s, tid);
  group_sync<GT>(bar);
}

// Passes NS0 .. P of a row (pass-major twiddle offset OFF of the first one).
template <int P, int E, int NS, int OFF, bool INV, int GT>
__device__ __forceinline__ void fft_passes(double2* s, int tid, const double2* tw, int bar);

__host__ __device__ constexpr int pass_radix(int p, int ns) { return p / ns >= 8 ? 8 : p / ns; }

// Entries of the pass-major twiddle table for a length-P row.
__host__ __device__ constexpr int twiddle_entries(int p) {
  int total = 0;
  for (int ns = 1; ns < p; ns *= pass_radix(p, ns))
    if (ns > 1) total += (pass_radix(p, ns) - 1) * ns;
  return total;
}

template <int P, int E, int NS, int OFF, bool INV, int GT>
__device__ __forceinline__ void fft_passes(double2* s, int tid, const double2* tw, int bar) {
  if constexpr (NS < P) {
    constexpr int R = pass_radix(P, NS);
    stockham_pass<P, E, R, NS, INV, GT>(s, tid, tw + OFF, bar);
    fft_passes<P, E, NS * R, OFF + (NS > 1 ? (R - 1) * NS : 0), INV, GT>(s, tid, tw, bar);
  }
}

// Full in-smem FFT of one padded row (P points, TR = P/E threads); input and
// output in natural order at s[smem_pad(i)]; `tw` = the pass-major table
// (forward signs; conjugated on the fly for the inverse; global or shared).
// Ends with a barrier over the row's threads (see group_sync).
template <int P, int E, bool INV, int GT = 0>
__device__ __forceinline__ void fft_row_smem(double2* s, int tid, const double2* tw, int bar = 0) {
  fft_passes<P, E, 1, 0, INV, GT>(s, tid, tw, bar);
}

// Ns of the last pass, and the pass-major table offset of the pass with Ns.
__host__ __device__ constexpr int last_pass_ns(int p) {
  int ns = 1;
  while (ns * pass_radix(p, ns) < p) ns *= pass_radix(p, ns);
  return ns;
}
__host__ __device__ constexpr int pass_tw_offset(int p, int ns_target) {
  int off = 0;
  for (int ns = 1; ns < ns_target; ns *= pass_radix(p, ns))
    if (ns > 1) off += (pass_radix(p, ns) - 1) * ns;
  return off;
}

// The passes with NS <= ns < NS_END (each ending with a row barrier).
template <int P, int E, int NS, int NS_END, bool INV, int GT, bool TWP = false>
__device__ __forceinline__ void mid_passes(double2* s, int tid, const double2* tw, int bar) {
  if constexpr (NS < NS_END) {
    constexpr int R = pass_radix(P, NS);
    stockham_pass<P, E, R, NS, INV, GT, TWP>(s, tid, tw + pass_tw_offset(P, NS), bar);
    mid_passes<P, E, NS * R, NS_END, INV, GT, TWP>(s, tid, tw, bar);
  }
}

// Ping-pong variant: each pass reads `src` and writes the other buffer, so the
// only barrier is the one after the store (the in-place pass needs a second
// one between its loads and its stores). Returns the buffer holding the
// result of the last pass run (a when NS == NS_END).
template <int P, int E, int R, int NS, bool INV, int GT, bool TWP = false>
__device__ __forceinline__ void stockham_pass_pp(const double2* src, double2* dst, int tid,
                                                 const double2* tw, int bar) {
  double2 v[E];
  pass_load<P, E, R>(v, src, tid);
  pass_compute<P, E, R, NS, INV, TWP>(v, tid, tw);
  pass_store<P, E, R, NS>(v, dst, tid);
  group_sync<GT>(bar);
}

template <int P, int E, int NS, int NS_END, bool INV, int GT, bool TWP = false>
__device__ __forceinline__ double2* mid_passes_pp(double2* a, double2* b, int tid,
                                                  const double2* tw, int bar) {
  if constexpr (NS < NS_END) {
    constexpr int R = pass_radix(P, NS);
    stockham_pass_pp<P, E, R, NS, INV, GT, TWP>(a, b, tid, tw + pass_tw_offset(P, NS), bar);
    return mid_passes_pp<P, E, NS * R, NS_END, INV, GT, TWP>(b, a, tid, tw, bar);
  } else {
    return a;
  }
}

// Device pass-major twiddle table for length 2^log2p (cached per device).
const double2* pass_twiddles(int log2p);

// Cooperative copy of a table into shared memory.
__device__ __forceinline__ void load_table(double2* dst, const double2* __restrict__ src, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
}

}  // namespace flb
