// Legendre <-> Chebyshev conversion (conversion.hpp:100-140) as an exact
// integer split GEMM on the tcgen05 tensor cores.
//
// Per parity class p the conversion is a triangular GEMM  C = A B  with
// A = the (N/2 x N/2) parity block of M (or of (m + 1/2) M^T for the IDLT)
// and B = the parity-p entries of the input columns. B200's fp64 tensor
// path (DMMA, leg2cheb.cu) peaks at ~37 TFLOP/s; its int8 tensor cores at
// ~4.5 POP/s. The split ("Ozaki") scheme runs the fp64 product on the int8
// units exactly:
//
//   row / column scaling:  A_ab = 2^{ea_a} sum_{i<S} a^(i)_ab 2^{-8(i+1)},
//                          B_bc = 2^{eb_c} sum_{j<S} b^(j)_bc 2^{-8(j+1)},
//   S = 7 signed 8-bit digits per operand (round-to-nearest splitting of the
//   scaled value, |value| < 1/4, exact in fp64; a +128 digit is carried into
//   the next higher one), so every digit product is exact (|.| <= 2^14) and
//   a K-sum of up to 7 of them fits int32 (7 * 2^14 * N/2 < 2^31 for
//   N <= 2^14):
//
//   C_ac = 2^{ea_a + eb_c} sum_{d < S} 2^{-8(d+2)} sum_{i+j=d} (a^(i) b^(j))_ac
//
// Pairs with i + j >= S are dropped: the largest is <= 2^14 2^{-8(S+2)} =
// 2^-58 of the row/column scales per term, the same order as an fp64 dot
// product's rounding (the 7-bit / 8-digit variant, -DFLB_OZ_DIGIT_BITS=7,
// drops at the same level with 36 pairs instead of 28: 9.9 vs 8.4 ms for
// C4's conversion).
//
// Kernel (persistent; output tiles of 128 rows x 64 columns of one parity;
// the default oz_gemm2_kernel pairs two SMs on 256-row tiles, cta_group::2):
//   warp 0     TMA producer: per 64-wide K block, the S slices of the A tile
//              (128 rows x 64 B) and of the B tile (64 or 32 columns x 64 B),
//              SWIZZLE_64B, into a ring of stages (3 x 70 KB for the pair
//              kernel with 7 digits)
//   warp 1     TMEM allocator and MMA issuer: 28 slice pairs x 2 K-steps of
//              tcgen05.mma.kind::i8 (M = 128/256, N = 64, K = 32) per stage,
//              fully unrolled, issued by one elected lane of the whole warp
//              (uniform operands); pair (i, j) accumulating into TMEM
//              accumulator d = i + j (S x 64 int32 columns)
//   warps 2-5  epilogue: tcgen05.ld of the S accumulators, exact int32 ->
//              fp64 scaled sum in registers, TMEM released to the next tile,
//              then row/column scales and the store (k = 2a + p)
// Only the K blocks on or above (forward) / below (transpose) the diagonal
// block are visited: the triangle costs half the square.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "common.cuh"
#include "l2c_ozaki.cuh"
#include "launch.cuh"

namespace flb {

namespace oz {
// Digit width: 8-bit digits (7 per operand, 28 pairs) by default; 7-bit
// digits (8 per operand, 36 pairs) with -DFLB_OZ_DIGIT_BITS=7.
#ifndef FLB_OZ_DIGIT_BITS
#define FLB_OZ_DIGIT_BITS 8
#endif
#ifndef FLB_OZ_TS1
#define FLB_OZ_TS1 1  // A operand from TMEM in the 1-SM kernel too
#endif
constexpr int DB = FLB_OZ_DIGIT_BITS;
constexpr int S = DB == 8 ? 7 : 8;  // digits per operand
constexpr int BM = 128;         // output rows per tile (TMEM lanes)
constexpr int BN = 64;          // output columns per tile
#ifndef FLB_OZ_BK
#define FLB_OZ_BK 64
#endif
#ifndef FLB_OZ_STAGES
#define FLB_OZ_STAGES 2
#endif
constexpr int BK = FLB_OZ_BK;   // K bytes per stage (32: SWIZZLE_32B rows, 64: SWIZZLE_64B)
constexpr int STAGES = FLB_OZ_STAGES;
constexpr int A_TILE = BM * BK;
constexpr int B_TILE = BN * BK;
constexpr int STAGE_BYTES = S * (A_TILE + B_TILE);
constexpr int THREADS = 192;                  // 6 warps
constexpr int EPI_THREADS = 128;              // warps 2-5
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
// kind::i8 instruction descriptor: D s32, A/B signed, K-major, N = 64, M = 128
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
}  // namespace oz

struct L2COzaki {
  size_t n = 0, r = 0;       // r = n / 2 rows (and K) per parity
  int mode = 0;              // kMode* (the product the A digits hold)
  int8_t* a = nullptr;       // [S][2][r][r] digits, K-major rows
  double* arow = nullptr;    // [2][r] row scales 2^ea
  CUtensorMap tmap_a;
};

namespace {

// ---- PTX helpers -------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Issued by a whole warp with warp-uniform operands (kept in uniform
// registers); one elected lane executes the MMA / commit. The same lane (the
// lowest active one) issues both, as tcgen05.commit tracks the issuing
// thread's MMAs.
__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_cp_128x256(uint32_t taddr, uint64_t sdesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(taddr),
      "l"(sdesc)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          bar)
      : "memory");
}
// K-major canonical layout of BK-byte rows swizzled over BK bytes (SWIZZLE_32B
// or _64B): 8-row groups 8 BK bytes apart (SBO), LBO unused.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  constexpr uint64_t layout = oz::BK == 64 ? 4 : 6;  // SWIZZLE_64B : SWIZZLE_32B
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) |
         ((uint64_t)(8 * oz::BK / 16) << 32) | (1ull << 46) /*sm100 version*/ | (layout << 61);
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- digit splitting ---------------------------------------------------
// Scale exponent e with max * 2^-e < 1/2 (7-bit digits) or < 1/4 (8-bit
// digits: the top digit keeps room for a carry); 0 for max = 0.
__device__ __forceinline__ int split_exp(double mx) {
  if (!(mx > 0.0)) return 0;
  int e;
  frexp(mx, &e);  // mx = m 2^e, m in [0.5, 1)
  return e + (oz::DB == 8 ? 2 : 1);
}
// Digits of r = x 2^-e: r = sum_j d_j 2^{-DB(j+1)} + O(2^{-DB S - 1}).
// rint(t) by the 1.5 * 2^52 shifter: t + M rounds to nearest even in the
// FP64 adder and the integer sits in the low mantissa bits (no F2I). Each
// residual is in [-1/2, 1/2], so a digit is in [-2^{DB-1}, 2^{DB-1}]: for
// DB = 7 that fits int8 as is; for DB = 8 a digit of +128 becomes -128 with
// a carry into the next higher digit (the value is unchanged; the top digit,
// |d_0| <= 64, absorbs any carry chain).
__device__ __forceinline__ void split_digits(double x, int e, int8_t (&d)[oz::S]) {
  constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
  constexpr double kRadix = oz::DB == 8 ? 256.0 : 128.0;
  double r = ldexp(x, -e);
  int di[oz::S];
#pragma unroll
  for (int j = 0; j < oz::S; ++j) {
    const double t = r * kRadix;
    const double y = t + kShift;
    di[j] = __double2loint(y);
    r = t - (y - kShift);
  }
  if constexpr (oz::DB == 8) {
#pragma unroll
    for (int j = oz::S - 1; j > 0; --j)
      if (di[j] == 128) {
        di[j] = -128;
        ++di[j - 1];
      }
  }
#pragma unroll
  for (int j = 0; j < oz::S; ++j) d[j] = (int8_t)di[j];
}

// Entry of the parity-p block: forward A[a][b] = pref_{2a+p} s_{b-a} s_{a+b+p}
// (b >= a); transpose A[b][a'] = sc_{2b+p} pref_{2a'+p} s_{b-a'} s_{a'+b+p} (a' <= b).
__device__ __forceinline__ double block_entry(const double* __restrict__ s, int transpose,
                                              int scale_half, int p, size_t row, size_t col) {
  size_t a, b;
  if (!transpose) {
    a = row, b = col;
  } else {
    a = col, b = row;
  }
  if (b < a) return 0.0;
  const double pref = (2 * a + p) == 0 ? 1.0 : 2.0;
  double v = pref * (s[b - a] * s[a + b + p]);
  if (transpose && scale_half) v *= (double)(2 * b + p) + 0.5;
  return v;
}

// One CTA per (parity, row): row scale and the S digit rows of A.
__global__ void __launch_bounds__(256) oz_split_a_kernel(const double* __restrict__ s, size_t r,
                                                         int transpose, int scale_half,
                                                         int8_t* __restrict__ a,
                                                         double* __restrict__ arow) {
  const int p = blockIdx.y;
  const size_t row = blockIdx.x;
  __shared__ double red[8];
  __shared__ int e_sh;
  double mx = 0.0;
  for (size_t c = threadIdx.x; c < r; c += blockDim.x)
    mx = fmax(mx, fabs(block_entry(s, transpose, scale_half, p, row, c)));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    e_sh = split_exp(m);
    arow[p * r + row] = ldexp(1.0, e_sh);
  }
  __syncthreads();
  const int e = e_sh;
  for (size_t c = threadIdx.x; c < r; c += blockDim.x) {
    int8_t d[oz::S];
    split_digits(block_entry(s, transpose, scale_half, p, row, c), e, d);
#pragma unroll
    for (int j = 0; j < oz::S; ++j) a[((size_t)(j * 2 + p) * r + row) * r + c] = d[j];
  }
}

// One CTA of n/EPT threads per input column (each thread one EPT-entry chunk,
// held in registers between the max reduction and the split): per-parity
// scales and the S digit slices, de-interleaved by parity ([S][2][cols][r]).
// EPT = 8 (n <= 8192: twice the resident warps of EPT = 16, so one CTA's
// reduction overlaps another's loads) or 16.
// A non-finite column gets a NaN scale so the product column comes out NaN
// (the NDCT input check reports it).
template <int EPT>
__global__ void __launch_bounds__(1024) oz_split_b_kernel(const double* __restrict__ in, size_t n,
                                                          size_t ld, size_t cols,
                                                          int8_t* __restrict__ b,
                                                          double* __restrict__ bcol,
                                                          int* nonfinite) {
  using W = typename std::conditional<EPT == 16, uint64_t, uint32_t>::type;  // EPT/2 digits
  constexpr int H = EPT / 2;
  const size_t col = blockIdx.x;
  const size_t r = n / 2;
  const size_t c = threadIdx.x;  // chunk: entries EPT c .. EPT c + EPT - 1
  __shared__ double red[2][32];
  __shared__ int e_sh[2];
  __shared__ int bad_sh;
  if (threadIdx.x == 0) bad_sh = 0;
  const double2* q = reinterpret_cast<const double2*>(in + col * ld + EPT * c);
  double2 v[H];
#pragma unroll
  for (int i = 0; i < H; ++i) v[i] = __ldcs(q + i);  // streamed: read once
  double mx0 = 0.0, mx1 = 0.0;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    bad |= !isfinite(v[i].x) || !isfinite(v[i].y);
    mx0 = fmax(mx0, fabs(v[i].x));
    mx1 = fmax(mx1, fabs(v[i].y));
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx0 = fmax(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = fmax(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  __syncthreads();
  if (bad) atomicOr(&bad_sh, 1);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = mx0;
    red[1][threadIdx.x >> 5] = mx1;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[threadIdx.x][w]);
    e_sh[threadIdx.x] = split_exp(m);
    bcol[threadIdx.x * cols + col] = bad_sh ? __longlong_as_double(0x7ff8000000000000ll)
                                            : ldexp(1.0, e_sh[threadIdx.x]);
    if (bad_sh && nonfinite && threadIdx.x == 0) atomicOr(nonfinite, 1);
  }
  __syncthreads();
  const int e0 = e_sh[0], e1 = e_sh[1];
  W w0[oz::S], w1[oz::S];
#pragma unroll
  for (int j = 0; j < oz::S; ++j) w0[j] = w1[j] = 0;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    int8_t d0[oz::S], d1[oz::S];
    split_digits(isfinite(v[i].x) ? v[i].x : 0.0, e0, d0);
    split_digits(isfinite(v[i].y) ? v[i].y : 0.0, e1, d1);
#pragma unroll
    for (int j = 0; j < oz::S; ++j) {
      w0[j] |= (W)(uint8_t)d0[j] << (8 * i);
      w1[j] |= (W)(uint8_t)d1[j] << (8 * i);
    }
  }
#pragma unroll
  for (int j = 0; j < oz::S; ++j) {
    *reinterpret_cast<W*>(b + ((size_t)(j * 2 + 0) * cols + col) * r + H * c) = w0[j];
    *reinterpret_cast<W*>(b + ((size_t)(j * 2 + 1) * cols + col) * r + H * c) = w1[j];
  }
}

// ---- the direct (dense) Legendre product ----------------------------------
// Plan-time table P_n(x_k), k < N/2, n < N, at the angles the reference
// evaluates: theta_k = theta*_kind(k) + delta_k (its exact grid angle plus the
// fp64 node offset, ndct.hpp:98-117 / quadrature.hpp:147-158), in
// double-double: the angle, cos by Taylor series at theta/64 and six double
// angle steps, and the three-term recurrence (oracle.hpp:19-48's order
// restated in dd), each entry rounded once to fp64. Layout [n][k] (the
// threads of a warp are consecutive nodes).
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd dd_two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_fast(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = dd_two_sum(a.hi, b.hi);
  const dd t = dd_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = dd_fast(s.hi, s.lo);
  s.lo += t.lo;
  return dd_fast(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return dd_fast(p, e);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  const double p = a.hi * b;
  double e = fma(a.hi, b, -p);
  e += a.lo * b;
  return dd_fast(p, e);
}
__device__ __forceinline__ dd dd_div_d(dd a, double b) {
  const double q1 = a.hi / b;
  const double p = q1 * b, pe = fma(q1, b, -p);
  double r = (a.hi - p) - pe + a.lo;
  return dd_fast(q1, r / b);
}

__global__ void legendre_table_kernel(size_t n, int kind, const double* __restrict__ delta,
                                      double* __restrict__ table) {
  const size_t r = n / 2;
  const size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (k >= r) return;
  const dd pi = {kPiHi, kPiLo};
  // theta*_k: (4k + 3) pi / (4N + 2) (chebstar) or (2k + 1) pi / (2N) (cheb1)
  dd th = kind == FL_CHEBSTAR ? dd_div_d(dd_mul_d(pi, 4.0 * (double)k + 3.0), 4.0 * (double)n + 2.0)
                              : dd_div_d(dd_mul_d(pi, 2.0 * (double)k + 1.0), 2.0 * (double)n);
  th = dd_add(th, dd{delta[k], 0.0});
  // cos / sin of theta / 64 by their Taylor series (|t| < 0.025: 10 terms
  // reach 1e-40), then six double-angle steps
  const dd t = {ldexp(th.hi, -6), ldexp(th.lo, -6)};
  const dd t2 = dd_mul(t, t);
  dd c = {1.0, 0.0}, sn = t, tc = {1.0, 0.0}, ts = t;
  for (int i = 1; i <= 10; ++i) {
    tc = dd_div_d(dd_mul(tc, t2), -(double)((2 * i - 1) * (2 * i)));
    ts = dd_div_d(dd_mul(ts, t2), -(double)((2 * i) * (2 * i + 1)));
    c = dd_add(c, tc);
    sn = dd_add(sn, ts);
  }
  for (int i = 0; i < 6; ++i) {
    const dd c2 = dd_add(dd_mul(c, c), dd_mul(dd{-sn.hi, -sn.lo}, sn));
    sn = dd_mul_d(dd_mul(sn, c), 2.0);
    c = c2;
  }
  const dd x = c;
  // P_0 = 1, P_1 = x, (m + 1) P_{m+1} = (2m + 1) x P_m - m P_{m-1}
  dd pm1 = {1.0, 0.0}, pm = x;
  table[k] = 1.0;
  if (n > 1) table[r + k] = x.hi;
  for (size_t m = 1; m + 1 < n; ++m) {
    const dd a = dd_mul_d(dd_mul(x, pm), 2.0 * (double)m + 1.0);
    const dd b = dd_mul_d(pm1, -(double)m);
    const dd nx = dd_div_d(dd_add(a, b), (double)(m + 1));
    pm1 = pm;
    pm = nx;
    table[(m + 1) * r + k] = pm.hi;
  }
}

// Entry of the dense parity-p block (table[n][k] = P_n(x_k)).
__device__ __forceinline__ double dense_entry(const double* __restrict__ table, size_t r, int idlt,
                                              int p, size_t row, size_t col) {
  if (!idlt) return table[(2 * col + p) * r + row];  // P_{2b+p}(x_a)
  const size_t deg = 2 * row + p;
  return ((double)deg + 0.5) * table[deg * r + col];  // (n + 1/2) P_n(x_b)
}

// One CTA per (parity, row): row scale and the S digit rows of the dense A.
__global__ void __launch_bounds__(256) oz_split_a_dense_kernel(const double* __restrict__ table,
                                                               size_t r, int idlt,
                                                               int8_t* __restrict__ a,
                                                               double* __restrict__ arow) {
  const int p = blockIdx.y;
  const size_t row = blockIdx.x;
  __shared__ double red[8];
  __shared__ int e_sh;
  double mx = 0.0;
  for (size_t c = threadIdx.x; c < r; c += blockDim.x)
    mx = fmax(mx, fabs(dense_entry(table, r, idlt, p, row, c)));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    e_sh = split_exp(m);
    arow[p * r + row] = ldexp(1.0, e_sh);
  }
  __syncthreads();
  const int e = e_sh;
  for (size_t c = threadIdx.x; c < r; c += blockDim.x) {
    int8_t d[oz::S];
    split_digits(dense_entry(table, r, idlt, p, row, c), e, d);
#pragma unroll
    for (int j = 0; j < oz::S; ++j) a[((size_t)(j * 2 + p) * r + row) * r + c] = d[j];
  }
}

// The direct IDLT's B operand, one CTA of r / H threads per column: entries
// b = t + i T (i < H) of u_p[b] = w_b (f_b + (-1)^p f_{N-1-b}), per-parity
// scales and the S digit slices ([S][2][cols][r], as oz_split_b_kernel).
template <int H>
__global__ void __launch_bounds__(1024) oz_split_b_sym_kernel(const double* __restrict__ in,
                                                              size_t n, size_t ld, size_t cols,
                                                              const double* __restrict__ w,
                                                              int8_t* __restrict__ b,
                                                              double* __restrict__ bcol,
                                                              int* nonfinite) {
  const size_t col = blockIdx.x;
  const size_t r = n / 2;
  const size_t T = blockDim.x;
  const size_t t = threadIdx.x;
  __shared__ double red[2][32];
  __shared__ int e_sh[2];
  __shared__ int bad_sh;
  if (threadIdx.x == 0) bad_sh = 0;
  const double* f = in + col * ld;
  double u0[H], u1[H];
  double mx0 = 0.0, mx1 = 0.0;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const size_t bi = t + i * T;
    const double wv = w[bi];
    const double fa = __ldcs(f + bi), fb = __ldcs(f + (n - 1 - bi));
    const double ga = wv * fa, gb = wv * fb;  // the weighted values (transforms.hpp:59)
    bad |= !isfinite(ga) || !isfinite(gb);
    u0[i] = ga + gb;
    u1[i] = ga - gb;
    mx0 = fmax(mx0, fabs(u0[i]));
    mx1 = fmax(mx1, fabs(u1[i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx0 = fmax(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = fmax(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  __syncthreads();
  if (bad) atomicOr(&bad_sh, 1);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = mx0;
    red[1][threadIdx.x >> 5] = mx1;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double m = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) m = fmax(m, red[threadIdx.x][q]);
    e_sh[threadIdx.x] = split_exp(m);
    bcol[threadIdx.x * cols + col] = bad_sh ? __longlong_as_double(0x7ff8000000000000ll)
                                            : ldexp(1.0, e_sh[threadIdx.x]);
    if (bad_sh && nonfinite && threadIdx.x == 0) atomicOr(nonfinite, 1);
  }
  __syncthreads();
  const int e0 = e_sh[0], e1 = e_sh[1];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const size_t bi = t + i * T;
    int8_t d0[oz::S], d1[oz::S];
    split_digits(isfinite(u0[i]) ? u0[i] : 0.0, e0, d0);
    split_digits(isfinite(u1[i]) ? u1[i] : 0.0, e1, d1);
#pragma unroll
    for (int j = 0; j < oz::S; ++j) {
      b[((size_t)(j * 2 + 0) * cols + col) * r + bi] = d0[j];
      b[((size_t)(j * 2 + 1) * cols + col) * r + bi] = d1[j];
    }
  }
}

// ---- the split GEMM ------------------------------------------------------
// Products the GEMM kernels compute (per parity p, rows a < r = N/2, K = r):
//   kModeTri / kModeTriT : the conversion M (upper-triangular parity blocks)
//                          or (m + 1/2) M^T (lower); output row 2a + p
//   kModeDenseDlt        : the direct DLT, A_p[a][b] = P_{2b+p}(x_a) (node a,
//                          degree 2b + p): E = A_0 c_even, O = A_1 c_odd, and
//                          f_a = E_a + O_a, f_{N-1-a} = E_a - O_a
//                          (P_n(-x) = (-1)^n P_n(x), x_{N-1-a} = -x_a)
//   kModeDenseIdlt       : the direct IDLT, A_p[a][b] = (n + 1/2) P_n(x_b),
//                          n = 2a + p, against u_p[b] = w_b (f_b + (-1)^p
//                          f_{N-1-b}); output row 2a + p
enum { kModeTri = 0, kModeTriT = 1, kModeDenseDlt = 2, kModeDenseIdlt = 3 };

// Epilogue store of one output row (a = tile row) over the tile's BN columns.
// Dense DLT: the parity-0 tile stores E_a at row a; the parity-1 tile of the
// same unit runs next on the same thread, reads E_a back (its own store, L2)
// and writes f_a = E_a + O_a and f_{N-1-a} = E_a - O_a.
__device__ __forceinline__ void store_tile(double* __restrict__ out, const double* acc,
                                           double ascale, const double* __restrict__ bcol,
                                           int mode, int p, size_t a, size_t cb, size_t r,
                                           size_t cols, size_t ld) {
  using namespace oz;
  if (mode == kModeDenseDlt) {
    if (p == 0) {
#pragma unroll
      for (int c = 0; c < BN; ++c) {
        const size_t col = cb * BN + c;
        if (col < cols) out[col * ld + a] = (acc[c] * ascale) * bcol[col];
      }
      return;
    }
    // E back in chunks: a chunk's loads are issued together, before its
    // stores (the compiler cannot move a load across a possibly aliasing
    // store, so a per-column load/store loop would serialise 64 L2 trips)
    constexpr int CH = 16;
#pragma unroll
    for (int c0 = 0; c0 < BN; c0 += CH) {
      double e[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const size_t col = cb * BN + c0 + i;
        e[i] = col < cols ? __ldcg(out + col * ld + a) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const size_t col = cb * BN + c0 + i;
        if (col >= cols) continue;
        const double v = (acc[c0 + i] * ascale) * bcol[cols + col];
        out[col * ld + a] = e[i] + v;
        out[col * ld + (2 * r - 1 - a)] = e[i] - v;
      }
    }
    return;
  }
  const size_t k = 2 * a + p;  // output row (interleaved parities)
#pragma unroll
  for (int c = 0; c < BN; ++c) {
    const size_t col = cb * BN + c;
    if (col < cols) out[col * ld + k] = (acc[c] * ascale) * bcol[(size_t)p * cols + col];
  }
}

// Persistent: CTA b takes tiles b, b + grid, ... (consecutive CTAs share a
// column block, so the B digits are reused from L2). The smem ring and its
// phases run continuously across tiles; the epilogue drains the 8 TMEM
// accumulators into fp64 registers, releases TMEM (tmem_empty) so the next
// tile's MMAs start, then scales and stores.
__global__ void __launch_bounds__(oz::THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b, const double* __restrict__ arow,
                   const double* __restrict__ bcol, double* __restrict__ out, size_t r,
                   size_t cols, size_t ld, int mode, size_t ntiles) {
  using namespace oz;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  // bars[0, STAGES) full, [STAGES, 2 STAGES) empty, [2 STAGES] tmem_full, [2 STAGES + 1] tmem_empty
  uint64_t* full_b = bars;
  uint64_t* empty_b = bars + STAGES;
  uint64_t* tfull_b = bars + 2 * STAGES;
  uint64_t* tempty_b = bars + 2 * STAGES + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t rb_count = r / BM;
  const int transpose = mode == kModeTriT;
  auto tile_coords = [&](size_t tile, size_t& cb, int& p, size_t& rb, int& kb_lo, int& nk) {
    cb = tile / (2 * rb_count);
    p = (int)(tile % 2);
    rb = (tile / 2) % rb_count;
    // K blocks (of BK) with nonzero entries: on/above (forward) or on/below
    // (transpose) the diagonal block; all of them for the dense products
    kb_lo = (transpose || mode >= kModeDenseDlt) ? 0 : (int)(rb * (BM / BK));
    const int kb_hi = mode >= kModeDenseDlt ? (int)(r / BK)
                      : transpose         ? (int)((rb + 1) * (BM / BK))
                                          : (int)(r / BK);
    nk = kb_hi - kb_lo;
  };
  // units of (column block, row block), both parities back to back on the
  // same CTA (the dense DLT's epilogue combines them)
  const size_t units = ntiles / 2;
  auto tile_of = [&](size_t i, size_t& tile) -> bool {
    const size_t u = blockIdx.x + (i >> 1) * gridDim.x;
    tile = 2 * u + (i & 1);
    return u < units;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * STAGES + 1; ++i) mbar_init(smem_u32(&bars[i]), 1);
    mbar_init(smem_u32(tempty_b), EPI_THREADS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      uint32_t it = 0;
      size_t tile;
      for (size_t ti = 0; tile_of(ti, tile); ++ti) {
        size_t cb, rb;
        int p, kb_lo, nk;
        tile_coords(tile, cb, p, rb, kb_lo, nk);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t st = it % STAGES, ph = (it / STAGES) & 1u;
          mbar_wait(smem_u32(&empty_b[st]), ph ^ 1u);
          const uint32_t full = smem_u32(&full_b[st]);
          mbar_expect_tx(full, STAGE_BYTES);
          uint8_t* sa = smem + st * STAGE_BYTES;
          uint8_t* sb = sa + S * A_TILE;
          const int k0 = (kb_lo + kb) * BK;
          for (int i = 0; i < S; ++i) {
            tma_load_3d(smem_u32(sa + i * A_TILE), &tmap_a, full, k0, (int)(rb * BM), i * 2 + p);
            tma_load_3d(smem_u32(sb + i * B_TILE), &tmap_b, full, k0, (int)(cb * BN), i * 2 + p);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // MMA issuer: the whole warp, one elected lane issues
      uint32_t it = 0, t = 0, aslot = 0;
      (void)aslot;
      size_t tile;
      for (size_t ti = 0; tile_of(ti, tile); ++ti, ++t) {
        size_t cb, rb;
        int p, kb_lo, nk;
        tile_coords(tile, cb, p, rb, kb_lo, nk);
        mbar_wait(smem_u32(tempty_b), (t & 1u) ^ 1u);  // epilogue drained the accumulators
        tc_fence_after();
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t st = it % STAGES, ph = (it / STAGES) & 1u;
          mbar_wait(smem_u32(&full_b[st]), ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + st * STAGE_BYTES);
          const uint64_t ad0 = smem_desc(sa), bd0 = smem_desc(sa + S * A_TILE);
          const uint32_t first = kb == 0 ? 0u : 1u;
          if constexpr (FLB_OZ_TS1 && S * BN + 64 <= 512) {
            // A digit tiles through TMEM (TS form), as in oz_gemm2_kernel
            tc_cp_128x256(tmem + (uint32_t)(S * BN + (aslot & 7u) * 8u), ad0);  // copy ahead
#pragma unroll
            for (int ks = 0; ks < BK / 32; ++ks) {
#pragma unroll
              for (int i = 0; i < S; ++i, ++aslot) {
                const uint32_t ta = tmem + (uint32_t)(S * BN + (aslot & 7u) * 8u);
                if (i + 1 < S || ks + 1 < BK / 32) {
                  const int ni = i + 1 < S ? i + 1 : 0, nks = i + 1 < S ? ks : ks + 1;
                  tc_cp_128x256(tmem + (uint32_t)(S * BN + ((aslot + 1) & 7u) * 8u),
                                ad0 + (uint64_t)((ni * A_TILE + nks * 32) >> 4));
                }
#pragma unroll
                for (int j = 0; i + j < S; ++j) {
                  const uint64_t bd = bd0 + (uint64_t)((j * B_TILE + ks * 32) >> 4);
                  tc_mma_i8_ts(tmem + (uint32_t)((i + j) * BN), ta, bd, IDESC,
                               (ks > 0 || i > 0) ? 1u : first);
                }
              }
            }
          } else {
          // fully unrolled: each MMA is a descriptor add and the UTCIMMA
#pragma unroll
          for (int i = 0; i < S; ++i) {
#pragma unroll
            for (int j = 0; i + j < S; ++j) {
#pragma unroll
              for (int ks = 0; ks < BK / 32; ++ks) {
                const uint64_t ad = ad0 + (uint64_t)((i * A_TILE + ks * 32) >> 4);
                const uint64_t bd = bd0 + (uint64_t)((j * B_TILE + ks * 32) >> 4);
                tc_mma_i8(tmem + (uint32_t)((i + j) * BN), ad, bd, IDESC,
                          (ks > 0 || i > 0) ? 1u : first);
              }
            }
          }
          }
          tc_commit_elect(smem_u32(&empty_b[st]));  // frees the stage when these MMAs retire
        }
        tc_commit_elect(smem_u32(tfull_b));  // accumulators complete
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +32 (one output row per thread)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    uint32_t t = 0;
    size_t tile;
    for (size_t ti = 0; tile_of(ti, tile); ++ti, ++t) {
      size_t cb, rb;
      int p, kb_lo, nk;
      tile_coords(tile, cb, p, rb, kb_lo, nk);
      mbar_wait(smem_u32(tfull_b), t & 1u);
      tc_fence_after();
      double acc[BN];
#pragma unroll
      for (int c = 0; c < BN; ++c) acc[c] = 0.0;
      // least significant accumulator first
#pragma unroll 1
      for (int d = S - 1; d >= 0; --d) {
        // exact S_d 2^{-DB(d+2)} without the int->fp64 conversion unit: the
        // biased integer becomes the low mantissa bits of a double whose ulp
        // is 2^{-DB(d+2)}; subtracting the bias constant is exact
        const int sh = DB * (d + 2);
        const int hi_word = (1075 - sh) << 20;
        const double bias = ldexp(1.0, 52 - sh) + ldexp(1.0, 31 - sh);
        uint32_t v[BN / 32][32];  // both halves in flight before one wait
#pragma unroll
        for (int h = 0; h < BN / 32; ++h)
          tmem_ld32_nowait(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(d * BN + h * 32), v[h]);
        tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < BN / 32; ++h)
#pragma unroll
          for (int c = 0; c < 32; ++c)
            acc[h * 32 + c] += __hiloint2double(hi_word, (int)(v[h][c] ^ 0x80000000u)) - bias;
      }
      tc_fence_before();
      mbar_arrive(smem_u32(tempty_b));  // TMEM free for the next tile
      const double ascale = arow[(size_t)p * r + rb * BM + row];
      store_tile(out, acc, ascale, bcol, mode, p, rb * BM + row, cb, r, cols, ld);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ---- the split GEMM on SM pairs (cta_group::2) -----------------------------
// A cluster of two CTAs on one TPC computes a 256 x 64 output tile (two
// adjacent 128-row blocks of one parity): each CTA stages its own 128 A rows
// and HALF of the B tile (32 columns) per K block, the leader issues
// tcgen05.mma.cta_group::2 (M = 256, N = 64) which reads both CTAs' shared
// memory, and each CTA's TMEM receives its 128 rows of the 8 accumulators.
// Per SM the tensor core then reads 4 KiB of A + 1 KiB of B per 32-clock MMA
// instead of 4 + 2 KiB: the shared-memory operand bound of the 1-SM kernel
// (64 % of the int8 peak at N = 64) rises to ~80 %.
#ifndef FLB_OZ_TS
#define FLB_OZ_TS 1  // A operand from TMEM in the pair kernel (needs S * 64 + 64 <= 512 columns)
#endif
namespace oz2 {
constexpr bool TS = FLB_OZ_TS && oz::S * oz::BN + 64 <= 512;
// 0 (default): the next tile's MMAs wait until the whole TMEM is drained;
// 1: the first K step is issued by accumulator in the drain order (all A
// digits copied first); 2: the epilogue drains the most significant
// accumulator first and the first K step's MMAs, in their usual order, wait
// for their own accumulator only. Both overlaps measured slower (C4 DLT 12.9
// and 13.2 vs 12.6 ms on one box): seven mbarrier waits in the single MMA
// issuing thread cost more than the drain they hide.
#ifndef FLB_OZ_ACC_OVERLAP
#define FLB_OZ_ACC_OVERLAP 0
#endif
constexpr int ACC_OVERLAP = TS ? FLB_OZ_ACC_OVERLAP : 0;
constexpr int A_TILE = oz::BM * oz::BK;            // 128 rows
constexpr int B_TILE = (oz::BN / 2) * oz::BK;      // 32 columns: this CTA's half
constexpr int STAGE_BYTES = oz::S * (A_TILE + B_TILE);
#ifndef FLB_OZ2_STAGES
#define FLB_OZ2_STAGES (oz::S == 7 ? 3 : 2)  // 3 x 70 KB fit with 7 digits
#endif
constexpr int STAGES = FLB_OZ2_STAGES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(oz::BN >> 3) << 17) |
                           ((uint32_t)(256 >> 4) << 24);
}  // namespace oz2

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA into this CTA's smem, completion counted on an mbarrier of the pair
// (the leader's), with an L2 eviction-priority hint: the A digits (the plan's
// matrix, re-read by every column block) evict last, the streamed B digits
// first.
#ifndef FLB_OZ_L2HINT
#define FLB_OZ_L2HINT 0  // measured slower (C4 DLT 13.1 vs 12.2 ms): B is shared by the 8 row-pair clusters
#endif
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map,
                                                 uint32_t cluster_bar, int c0, int c1, int c2,
                                                 uint64_t policy) {
#if FLB_OZ_L2HINT
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(cluster_bar), "r"(c0), "r"(c1), "r"(c2),
      "l"(policy)
      : "memory");
#else
  (void)policy;
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(cluster_bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
#endif
}
__device__ __forceinline__ void tc2_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// TS form: A (this CTA's 128 rows) from TMEM, B from shared memory.
__device__ __forceinline__ void tc2_mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// smem (128 rows x 32 bytes, the operand descriptor's layout) -> TMEM
// (128 lanes x 8 columns) in both CTAs of the pair; ordered with the MMAs.
__device__ __forceinline__ void tc2_cp_128x256(uint32_t taddr, uint64_t sdesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.cp.cta_group::2.128x256b [%0], %1;\n\t}" ::"r"(taddr),
      "l"(sdesc)
      : "memory");
}
// Arrive on the barrier at this offset in BOTH CTAs of the pair once the
// issuing thread's MMAs retire.
__device__ __forceinline__ void tc2_commit_both(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(oz::THREADS, 1)
    oz_gemm2_kernel(const __grid_constant__ CUtensorMap tmap_a,
                    const __grid_constant__ CUtensorMap tmap_b, const double* __restrict__ arow,
                    const double* __restrict__ bcol, double* __restrict__ out, size_t r,
                    size_t cols, size_t ld, int mode, size_t ntiles) {
  using namespace oz;
  using oz2::A_TILE;
  using oz2::B_TILE;
  using oz2::STAGE_BYTES;
  using oz2::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full_b = bars;                 // leader's are used (count 2: both producers)
  uint64_t* empty_b = bars + STAGES;       // each CTA's own (multicast commit)
  uint64_t* tfull_b = bars + 2 * STAGES;   // each CTA's own (multicast commit)
  uint64_t* tempty_b = bars + 2 * STAGES + 1;  // leader's (both epilogues arrive)
  // FLB_OZ_ACC_OVERLAP: one "drained" barrier per accumulator (leader's; one
  // arrival per epilogue warp of both CTAs), so the next tile's first MMAs
  // into accumulator d start as soon as d has been read out
  uint64_t* acc_b = bars + 2 * STAGES + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2 + S);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const size_t pairs = (r / BM) / 2;  // 256-row blocks
  const size_t cluster_id = blockIdx.x / 2, nclusters = gridDim.x / 2;
  const int transpose = mode == kModeTriT;
  auto tile_coords = [&](size_t tile, size_t& cb, int& p, size_t& rp, int& kb_lo, int& nk) {
    cb = tile / (2 * pairs);
    p = (int)(tile % 2);
    rp = (tile / 2) % pairs;
    // K blocks with nonzero entries for either 128-row block of the pair (all
    // of them for the dense products)
    kb_lo = (transpose || mode >= kModeDenseDlt) ? 0 : (int)(rp * 2 * (BM / BK));
    const int kb_hi = mode >= kModeDenseDlt ? (int)(r / BK)
                      : transpose         ? (int)((rp + 1) * 2 * (BM / BK))
                                          : (int)(r / BK);
    nk = kb_hi - kb_lo;
  };
  const size_t units = ntiles / 2;  // both parities of a unit back to back (see oz_gemm_kernel)
  auto tile_of = [&](size_t i, size_t& tile) -> bool {
    const size_t u = cluster_id + (i >> 1) * nclusters;
    tile = 2 * u + (i & 1);
    return u < units;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(smem_u32(&full_b[i]), 2);
      mbar_init(smem_u32(&empty_b[i]), 1);
    }
    mbar_init(smem_u32(tfull_b), 1);
    mbar_init(smem_u32(tempty_b), 2 * EPI_THREADS);
    for (int d = 0; d < S; ++d) mbar_init(smem_u32(&acc_b[d]), 2 * (EPI_THREADS / 32));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs)
      const uint64_t pol_a = l2_policy_evict_last(), pol_b = l2_policy_evict_first();
      uint32_t it = 0;
      size_t tile;
      for (size_t ti = 0; tile_of(ti, tile); ++ti) {
        size_t cb, rp;
        int p, kb_lo, nk;
        tile_coords(tile, cb, p, rp, kb_lo, nk);
        const int row0 = (int)((2 * rp + rank) * BM);
        const int col0 = (int)(cb * BN + rank * (BN / 2));
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t st = it % STAGES, ph = (it / STAGES) & 1u;
          mbar_wait(smem_u32(&empty_b[st]), ph ^ 1u);
          const uint32_t full_leader = map_to_rank(smem_u32(&full_b[st]), 0);
          if (leader)
            mbar_expect_tx(smem_u32(&full_b[st]), 2 * STAGE_BYTES);
          else
            mbar_arrive_remote(full_leader);
          uint8_t* sa = smem + st * STAGE_BYTES;
          uint8_t* sb = sa + S * A_TILE;
          const int k0 = (kb_lo + kb) * BK;
          for (int i = 0; i < S; ++i) {
            tma_load_3d_pair(smem_u32(sa + i * A_TILE), &tmap_a, full_leader, k0, row0, i * 2 + p,
                             pol_a);
            tma_load_3d_pair(smem_u32(sb + i * B_TILE), &tmap_b, full_leader, k0, col0, i * 2 + p,
                             pol_b);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // MMA issuer: the leader's whole warp, one elected lane issues
      uint32_t it = 0, t = 0, aslot = 0;
      (void)aslot;
      size_t tile;
      for (size_t ti = 0; tile_of(ti, tile); ++ti, ++t) {
        size_t cb, rp;
        int p, kb_lo, nk;
        tile_coords(tile, cb, p, rp, kb_lo, nk);
        if constexpr (!oz2::ACC_OVERLAP) {
          mbar_wait(smem_u32(tempty_b), (t & 1u) ^ 1u);  // both epilogues drained TMEM
          tc_fence_after();
        }
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t st = it % STAGES, ph = (it / STAGES) & 1u;
          mbar_wait(smem_u32(&full_b[st]), ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + st * STAGE_BYTES);
          const uint64_t ad0 = smem_desc(sa), bd0 = smem_desc(sa + S * A_TILE);
          const uint32_t first = kb == 0 ? 0u : 1u;
          if (oz2::ACC_OVERLAP == 1 && kb == 0) {
            // the tile's first K step, by accumulator in the epilogue's drain
            // order (least significant first): all S A-digit tiles into S
            // slots, then for d = S-1 .. 0 wait until both epilogues have read
            // accumulator d of the previous tile and issue the pairs
            // (i, d - i), the first one (i = 0) overwriting it
#pragma unroll
            for (int i = 0; i < S; ++i)
              tc2_cp_128x256(tmem + (uint32_t)(S * BN + ((aslot + i) & 7u) * 8u),
                             ad0 + (uint64_t)((i * A_TILE) >> 4));
#pragma unroll
            for (int d = S - 1; d >= 0; --d) {
              mbar_wait(smem_u32(&acc_b[d]), (t & 1u) ^ 1u);
              tc_fence_after();
#pragma unroll
              for (int i = 0; i <= d; ++i) {
                const uint64_t bd = bd0 + (uint64_t)(((d - i) * B_TILE) >> 4);
                tc2_mma_i8_ts(tmem + (uint32_t)(d * BN), tmem + (uint32_t)(S * BN + ((aslot + i) & 7u) * 8u),
                              bd, oz2::IDESC, i > 0 ? 1u : 0u);
              }
            }
            aslot += S;
            // the remaining K steps of this block in the usual order
            if constexpr (BK / 32 > 1) {
              tc2_cp_128x256(tmem + (uint32_t)(S * BN + (aslot & 7u) * 8u),
                             ad0 + (uint64_t)(32 >> 4));
#pragma unroll
              for (int ks = 1; ks < BK / 32; ++ks) {
#pragma unroll
                for (int i = 0; i < S; ++i, ++aslot) {
                  const uint32_t ta = tmem + (uint32_t)(S * BN + (aslot & 7u) * 8u);
                  if (i + 1 < S || ks + 1 < BK / 32) {
                    const int ni = i + 1 < S ? i + 1 : 0, nks = i + 1 < S ? ks : ks + 1;
                    tc2_cp_128x256(tmem + (uint32_t)(S * BN + ((aslot + 1) & 7u) * 8u),
                                   ad0 + (uint64_t)((ni * A_TILE + nks * 32) >> 4));
                  }
#pragma unroll
                  for (int j = 0; i + j < S; ++j) {
                    const uint64_t bd = bd0 + (uint64_t)((j * B_TILE + ks * 32) >> 4);
                    tc2_mma_i8_ts(tmem + (uint32_t)((i + j) * BN), ta, bd, oz2::IDESC, 1u);
                  }
                }
              }
            }
          } else if constexpr (oz2::TS) {
          if (oz2::ACC_OVERLAP == 2 && kb == 0) {
            // the tile's first K step: the (0, j) MMA overwrites accumulator j
            // once both epilogues have read it (drained 0 .. S-1, in this order)
            tc2_cp_128x256(tmem + (uint32_t)(S * BN + (aslot & 7u) * 8u), ad0);
            tc2_cp_128x256(tmem + (uint32_t)(S * BN + ((aslot + 1) & 7u) * 8u),
                           ad0 + (uint64_t)((A_TILE) >> 4));
#pragma unroll
            for (int j = 0; j < S; ++j) {
              mbar_wait(smem_u32(&acc_b[j]), (t & 1u) ^ 1u);
              tc_fence_after();
              tc2_mma_i8_ts(tmem + (uint32_t)(j * BN), tmem + (uint32_t)(S * BN + (aslot & 7u) * 8u),
                            bd0 + (uint64_t)((j * B_TILE) >> 4), oz2::IDESC, 0u);
            }
            ++aslot;
#pragma unroll
            for (int ks = 0; ks < BK / 32; ++ks) {
#pragma unroll
              for (int i = ks == 0 ? 1 : 0; i < S; ++i, ++aslot) {
                const uint32_t ta = tmem + (uint32_t)(S * BN + (aslot & 7u) * 8u);
                if ((i + 1 < S || ks + 1 < BK / 32) && !(ks == 0 && i == 0)) {
                  const int ni = i + 1 < S ? i + 1 : 0, nks = i + 1 < S ? ks : ks + 1;
                  tc2_cp_128x256(tmem + (uint32_t)(S * BN + ((aslot + 1) & 7u) * 8u),
                                 ad0 + (uint64_t)((ni * A_TILE + nks * 32) >> 4));
                }
#pragma unroll
                for (int j = 0; i + j < S; ++j) {
                  const uint64_t bd = bd0 + (uint64_t)((j * B_TILE + ks * 32) >> 4);
                  tc2_mma_i8_ts(tmem + (uint32_t)((i + j) * BN), ta, bd, oz2::IDESC, 1u);
                }
              }
            }
          } else {
          // A digit tiles through TMEM: each (K-step, digit) tile is copied
          // once into one of 8 rotating 8-column slots after the S x 64
          // accumulator columns and read there by its S - i MMAs (the copy
          // and the MMAs run in issue order, so a slot is rewritten only
          // after the MMAs issued before the copy have read it). Shared
          // memory then serves A once per tile instead of once per MMA.
          // each digit's copy is issued one digit ahead of its MMAs, so an
          // MMA never waits on the copy it reads (copy-then-MMA ran at 75 %
          // of the MMA rate in tools/tc_i8_peak.cu, copy-ahead at 86 %)
          tc2_cp_128x256(tmem + (uint32_t)(S * BN + (aslot & 7u) * 8u), ad0);
#pragma unroll
          for (int ks = 0; ks < BK / 32; ++ks) {
#pragma unroll
            for (int i = 0; i < S; ++i, ++aslot) {
              const uint32_t ta = tmem + (uint32_t)(S * BN + (aslot & 7u) * 8u);
              if (i + 1 < S || ks + 1 < BK / 32) {
                const int ni = i + 1 < S ? i + 1 : 0, nks = i + 1 < S ? ks : ks + 1;
                tc2_cp_128x256(tmem + (uint32_t)(S * BN + ((aslot + 1) & 7u) * 8u),
                               ad0 + (uint64_t)((ni * A_TILE + nks * 32) >> 4));
              }
#pragma unroll
              for (int j = 0; i + j < S; ++j) {
                const uint64_t bd = bd0 + (uint64_t)((j * B_TILE + ks * 32) >> 4);
                tc2_mma_i8_ts(tmem + (uint32_t)((i + j) * BN), ta, bd, oz2::IDESC,
                              (ks > 0 || i > 0) ? 1u : first);
              }
            }
          }
          }
          } else {
#pragma unroll
          for (int i = 0; i < S; ++i) {
#pragma unroll
            for (int j = 0; i + j < S; ++j) {
#pragma unroll
              for (int ks = 0; ks < BK / 32; ++ks) {
                const uint64_t ad = ad0 + (uint64_t)((i * A_TILE + ks * 32) >> 4);
                const uint64_t bd = bd0 + (uint64_t)((j * B_TILE + ks * 32) >> 4);
                tc2_mma_i8(tmem + (uint32_t)((i + j) * BN), ad, bd, oz2::IDESC,
                           (ks > 0 || i > 0) ? 1u : first);
              }
            }
          }
          }
          tc2_commit_both(smem_u32(&empty_b[st]));  // frees the stage in both CTAs
        }
        tc2_commit_both(smem_u32(tfull_b));  // accumulators complete in both CTAs
      }
    }
  } else {
    // epilogue (both CTAs): TMEM lanes = this CTA's 128 rows of the 256-row tile
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t tempty_leader = map_to_rank(smem_u32(tempty_b), 0);
    const uint32_t acc_leader = map_to_rank(smem_u32(acc_b), 0);
    uint32_t t = 0;
    size_t tile;
    for (size_t ti = 0; tile_of(ti, tile); ++ti, ++t) {
      size_t cb, rp;
      int p, kb_lo, nk;
      tile_coords(tile, cb, p, rp, kb_lo, nk);
      const size_t rb = 2 * rp + rank;
      mbar_wait(smem_u32(tfull_b), t & 1u);
      tc_fence_after();
      double acc[BN];
#pragma unroll
      for (int c = 0; c < BN; ++c) acc[c] = 0.0;
#pragma unroll 1
      for (int dd = S - 1; dd >= 0; --dd) {
        // (overlap 2: the most significant accumulator first, so the next
        // tile's first MMAs -- into accumulator 0 first -- can start)
        const int d = oz2::ACC_OVERLAP == 2 ? S - 1 - dd : dd;
        // exact S_d 2^{-DB(d+2)} without the int->fp64 conversion unit: the
        // biased integer becomes the low mantissa bits of a double whose ulp
        // is 2^{-DB(d+2)}; subtracting the bias constant is exact
        const int sh = DB * (d + 2);
        const int hi_word = (1075 - sh) << 20;
        const double bias = ldexp(1.0, 52 - sh) + ldexp(1.0, 31 - sh);
        uint32_t v[BN / 32][32];  // both halves in flight before one wait
#pragma unroll
        for (int h = 0; h < BN / 32; ++h)
          tmem_ld32_nowait(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(d * BN + h * 32), v[h]);
        tmem_wait_ld();
        if constexpr (oz2::ACC_OVERLAP) {  // accumulator d read out: the next tile may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(acc_leader + 8u * (uint32_t)d);
        }
#pragma unroll
        for (int h = 0; h < BN / 32; ++h)
#pragma unroll
          for (int c = 0; c < 32; ++c)
            acc[h * 32 + c] += __hiloint2double(hi_word, (int)(v[h][c] ^ 0x80000000u)) - bias;
      }
      tc_fence_before();
      if constexpr (!oz2::ACC_OVERLAP) mbar_arrive_remote(tempty_leader);  // TMEM free for the pair's next tile
      const double ascale = arow[(size_t)p * r + rb * BM + row];
      store_tile(out, acc, ascale, bcol, mode, p, rb * BM + row, cb, r, cols, ld);
    }
  }
  tc_fence_before();
  cluster_sync_all();  // the peer's smem / TMEM stay live until the leader is done
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    FLB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f)
      fail(FL_CUDA_ERROR, "l2c_ozaki: cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 3-D int8 map [z][rows][k] with a (BK x box_rows x 1) SWIZZLE_64B box.
CUtensorMap make_map(const int8_t* base, size_t k, size_t rows, size_t z, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)k, (cuuint64_t)rows, (cuuint64_t)z};
  cuuint64_t strides[2] = {(cuuint64_t)k, (cuuint64_t)(k * rows)};
  cuuint32_t box[3] = {(cuuint32_t)oz::BK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult res = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   oz::BK == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS) fail(FL_CUDA_ERROR, "l2c_ozaki: tensor map encode failed");
  return m;
}

}  // namespace

void launch_legendre_table(size_t n, int kind, const double* delta, double* table, cudaStream_t st) {
  const size_t r = n / 2;
  legendre_table_kernel<<<(unsigned)((r + 127) / 128), 128, 0, st>>>(n, kind, delta, table);
  note_launch("legendre_table_kernel");
}

bool l2c_ozaki_supported(size_t n) { return n % 256 == 0 && n >= 512 && n <= 16384; }

L2COzaki* l2c_ozaki_create(size_t n, const double* s, int transpose, int scale_half,
                           cudaStream_t st) {
  if (!l2c_ozaki_supported(n)) fail(FL_INVALID_ARGUMENT, "l2c_ozaki: unsupported size");
  auto* p = new L2COzaki;
  p->n = n;
  p->r = n / 2;
  p->mode = transpose;  // kModeTri / kModeTriT
  const size_t r = p->r;
  FLB_CUDA(cudaMalloc(&p->a, (size_t)oz::S * 2 * r * r));
  FLB_CUDA(cudaMalloc(&p->arow, 2 * r * sizeof(double)));
  oz_split_a_kernel<<<dim3((unsigned)r, 2), 256, 0, st>>>(s, r, transpose, scale_half, p->a,
                                                          p->arow);
  note_launch("oz_split_a_kernel");
  p->tmap_a = make_map(p->a, r, r, 2 * oz::S, oz::BM);
  return p;
}

void l2c_ozaki_destroy(L2COzaki* p) {
  if (!p) return;
  cudaFree(p->a);
  cudaFree(p->arow);
  delete p;
}

namespace {

// The split GEMM over prepared B digits ([S][2][cols][r]) and column scales.
void launch_gemm(const L2COzaki& p, const int8_t* b, const double* bcol, double* out, size_t cols,
                 size_t ld, cudaStream_t st) {
  const size_t r = p.r;
  const CUtensorMap tmap_b = make_map(b, r, cols, 2 * oz::S, oz::BN);
  // the attribute is per device context: set it on every call (the library
  // serves several devices in one process)
  FLB_CUDA(cudaFuncSetAttribute(oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                oz::SMEM));
#ifndef FLB_OZ_PAIR
#define FLB_OZ_PAIR 1
#endif
  if (FLB_OZ_PAIR && (r / oz::BM) % 2 == 0) {
    // SM pairs: tiles of 256 rows x 64 columns, B staged as two 32-column halves
    const CUtensorMap tmap_b2 = make_map(b, r, cols, 2 * oz::S, oz::BN / 2);
    FLB_CUDA(cudaFuncSetAttribute(oz_gemm2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  oz2::SMEM));
    const size_t tiles = 2 * (r / oz::BM / 2) * ((cols + oz::BN - 1) / oz::BN);
    const unsigned clusters = (unsigned)std::min<size_t>(tiles / 2, (size_t)sm_count() / 2);
    oz_gemm2_kernel<<<2 * clusters, oz::THREADS, oz2::SMEM, st>>>(
        p.tmap_a, tmap_b2, p.arow, bcol, out, r, cols, ld, p.mode, tiles);
    note_launch("oz_gemm2_kernel");
  } else {
    const size_t tiles = 2 * (r / oz::BM) * ((cols + oz::BN - 1) / oz::BN);
    const unsigned grid = (unsigned)std::min<size_t>(tiles / 2, (size_t)sm_count());
    oz_gemm_kernel<<<grid, oz::THREADS, oz::SMEM, st>>>(p.tmap_a, tmap_b, p.arow, bcol, out, r,
                                                         cols, ld, p.mode, tiles);
    note_launch("oz_gemm_kernel");
  }
}

}  // namespace

void l2c_ozaki_apply(const L2COzaki& p, const double* in, double* out, size_t cols, size_t ld,
                     cudaStream_t st) {
  if (cols == 0) return;
  const size_t n = p.n, r = p.r;
  // the digit split reads the columns as double2: a column start that is only
  // 8-byte aligned (odd stride, or a view at an odd element offset) goes
  // through a packed, aligned copy instead of faulting
  if ((reinterpret_cast<uintptr_t>(in) & 15) != 0 || (ld & 1) != 0) {
    double* packed = nullptr;
    FLB_CUDA(cudaMallocAsync(&packed, n * cols * sizeof(double), st));
    FLB_CUDA(cudaMemcpy2DAsync(packed, n * 8, in, ld * 8, n * 8, cols, cudaMemcpyDeviceToDevice,
                               st));
    if (ld == n) {
      l2c_ozaki_apply(p, packed, out, cols, n, st);
    } else {  // one stride serves both sides: the product goes through a stride-n scratch
      double* res = nullptr;
      FLB_CUDA(cudaMallocAsync(&res, n * cols * sizeof(double), st));
      l2c_ozaki_apply(p, packed, res, cols, n, st);
      FLB_CUDA(cudaMemcpy2DAsync(out, ld * 8, res, n * 8, n * 8, cols, cudaMemcpyDeviceToDevice,
                                 st));
      cudaFreeAsync(res, st);
    }
    cudaFreeAsync(packed, st);
    return;
  }
  int8_t* b = nullptr;
  double* bcol = nullptr;
  FLB_CUDA(cudaMallocAsync(&b, (size_t)oz::S * 2 * cols * r, st));
  FLB_CUDA(cudaMallocAsync(&bcol, 2 * cols * sizeof(double), st));
#ifndef FLB_OZ_SPLIT8_MAX
#define FLB_OZ_SPLIT8_MAX 8192  // largest N split with 8 entries per thread
#endif
  if (n <= FLB_OZ_SPLIT8_MAX)
    oz_split_b_kernel<8><<<(unsigned)cols, (unsigned)(n / 8), 0, st>>>(in, n, ld, cols, b, bcol,
                                                                      nullptr);
  else
    oz_split_b_kernel<16><<<(unsigned)cols, (unsigned)(n / 16), 0, st>>>(in, n, ld, cols, b, bcol,
                                                                        nullptr);
  note_launch("oz_split_b_kernel");
  launch_gemm(p, b, bcol, out, cols, ld, st);
  cudaFreeAsync(b, st);
  cudaFreeAsync(bcol, st);
}


L2COzaki* l2c_dense_create(size_t n, int kind, const double* delta, int idlt, cudaStream_t st) {
  if (!l2c_dense_supported(n)) fail(FL_INVALID_ARGUMENT, "l2c_dense: unsupported size");
  auto* p = new L2COzaki;
  p->n = n;
  p->r = n / 2;
  p->mode = idlt ? kModeDenseIdlt : kModeDenseDlt;
  const size_t r = p->r;
  double* table = nullptr;
  FLB_CUDA(cudaMallocAsync(&table, n * r * sizeof(double), st));
  legendre_table_kernel<<<(unsigned)((r + 127) / 128), 128, 0, st>>>(n, kind, delta, table);
  note_launch("legendre_table_kernel");
  FLB_CUDA(cudaMalloc(&p->a, (size_t)oz::S * 2 * r * r));
  FLB_CUDA(cudaMalloc(&p->arow, 2 * r * sizeof(double)));
  oz_split_a_dense_kernel<<<dim3((unsigned)r, 2), 256, 0, st>>>(table, r, idlt, p->a, p->arow);
  note_launch("oz_split_a_dense_kernel");
  cudaFreeAsync(table, st);
  p->tmap_a = make_map(p->a, r, r, 2 * oz::S, oz::BM);
  return p;
}

bool l2c_dense_supported(size_t n) { return l2c_ozaki_supported(n) && n <= kDenseMaxN; }

void l2c_dense_apply(const L2COzaki& p, const double* in, size_t ld_in, const double* w,
                     double* out, size_t ld_out, size_t cols, int* nonfinite, cudaStream_t st) {
  if (cols == 0) return;
  const size_t n = p.n, r = p.r;
  const bool idlt = p.mode == kModeDenseIdlt;
  if (!idlt && ((reinterpret_cast<uintptr_t>(in) & 15) != 0 || (ld_in & 1) != 0)) {
    // the DLT's digit split reads double2: pack a misaligned block first
    double* packed = nullptr;
    FLB_CUDA(cudaMallocAsync(&packed, n * cols * sizeof(double), st));
    FLB_CUDA(cudaMemcpy2DAsync(packed, n * 8, in, ld_in * 8, n * 8, cols,
                               cudaMemcpyDeviceToDevice, st));
    l2c_dense_apply(p, packed, n, w, out, ld_out, cols, nonfinite, st);
    cudaFreeAsync(packed, st);
    return;
  }
  int8_t* b = nullptr;
  double* bcol = nullptr;
  FLB_CUDA(cudaMallocAsync(&b, (size_t)oz::S * 2 * cols * r, st));
  FLB_CUDA(cudaMallocAsync(&bcol, 2 * cols * sizeof(double), st));
  if (idlt) {
    oz_split_b_sym_kernel<4><<<(unsigned)cols, (unsigned)(r / 4), 0, st>>>(in, n, ld_in, cols, w, b,
                                                                          bcol, nonfinite);
    note_launch("oz_split_b_sym_kernel");
  } else {
    oz_split_b_kernel<8><<<(unsigned)cols, (unsigned)(n / 8), 0, st>>>(in, n, ld_in, cols, b, bcol,
                                                                      nonfinite);
    note_launch("oz_split_b_kernel");
  }
  launch_gemm(p, b, bcol, out, cols, ld_out, st);
  cudaFreeAsync(b, st);
  cudaFreeAsync(bcol, st);
}

}  // namespace flb
