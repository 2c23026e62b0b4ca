// Shared device/host helpers for libfastleg_b200: status plumbing, launch
// checks, double-double arithmetic for the node kernel, exact angle reduction.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "fastleg_b200.h"

namespace flb {

constexpr double kPi = 3.14159265358979323846264338327950288;  // types.hpp:36
// pi as a double-double (hi + lo)
constexpr double kPiHi = 3.141592653589793116e+00;
constexpr double kPiLo = 1.224646799147353207e-16;

// Thrown inside the library, converted to fl_status at the C boundary.
struct Error {
  fl_status status;
  std::string message;
};

[[noreturn]] void fail(fl_status s, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define FLB_CUDA(call) ::flb::cuda_check((call), #call)
#define FLB_LAUNCH(what) ::flb::cuda_check(cudaGetLastError(), what)

inline int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// ---- double-double ----------------------------------------------------
struct dd {
  double hi, lo;
};

__host__ __device__ inline dd dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__host__ __device__ inline dd dd_quick(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ inline dd dd_two_prod(double a, double b) {
  const double p = a * b;
  return {p, __fma_rn(a, b, -p)};
}
__device__ inline dd dd_add(dd x, dd y) {
  dd s = dd_two_sum(x.hi, y.hi);
  dd t = dd_two_sum(x.lo, y.lo);
  s.lo += t.hi;
  s = dd_quick(s.hi, s.lo);
  s.lo += t.lo;
  return dd_quick(s.hi, s.lo);
}
__device__ inline dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__device__ inline dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
__device__ inline dd dd_add_d(dd x, double y) {
  dd s = dd_two_sum(x.hi, y);
  s.lo += x.lo;
  return dd_quick(s.hi, s.lo);
}
__device__ inline dd dd_mul(dd x, dd y) {
  dd p = dd_two_prod(x.hi, y.hi);
  p.lo = __fma_rn(x.hi, y.lo, p.lo);
  p.lo = __fma_rn(x.lo, y.hi, p.lo);
  return dd_quick(p.hi, p.lo);
}
__device__ inline dd dd_mul_d(dd x, double y) {
  dd p = dd_two_prod(x.hi, y);
  p.lo = __fma_rn(x.lo, y, p.lo);
  return dd_quick(p.hi, p.lo);
}
__device__ inline dd dd_div(dd x, dd y) {
  const double q1 = x.hi / y.hi;
  dd r = dd_sub(x, dd_mul_d(y, q1));
  const double q2 = r.hi / y.hi;
  r = dd_sub(r, dd_mul_d(y, q2));
  const double q3 = r.hi / y.hi;
  dd q = dd_quick(q1, q2);
  return dd_add_d(q, q3);
}
__device__ inline dd dd_div_d(dd x, double y) { return dd_div(x, dd{y, 0.0}); }
__device__ inline dd dd_sqrt(dd a) {
  if (a.hi <= 0.0) return {0.0, 0.0};
  const double x = 1.0 / sqrt(a.hi);
  const double ax = a.hi * x;
  dd axsq = dd_two_prod(ax, ax);
  const double diff = dd_sub(a, axsq).hi * (x * 0.5);
  return dd_two_sum(ax, diff);
}
// sin(t) for 0 <= t <= pi/4 by its Taylor series (error ~1e-33)
__device__ inline dd dd_sin_small(dd t) {
  const dd t2 = dd_mul(t, t);
  dd term = t, sum = t;
  for (int i = 1; i <= 16; ++i) {
    term = dd_mul(term, t2);
    term = dd_div_d(term, -(double)((2 * i) * (2 * i + 1)));
    sum = dd_add(sum, term);
    if (fabs(term.hi) < 1e-36 * fabs(sum.hi)) break;
  }
  return sum;
}

// ---- exact angle reduction ---------------------------------------------
// e^{i pi num / den} with num reduced modulo 2*den in integer arithmetic, so
// the phase is exact before the single rounding of the quotient.
__device__ inline double2 expi_pi_frac(uint64_t num, uint64_t den) {
  const uint64_t r = num % (2 * den);
  double s, c;
  sincospi((double)r / (double)den, &s, &c);
  return make_double2(c, s);
}

__device__ inline double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ inline double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

}  // namespace flb
