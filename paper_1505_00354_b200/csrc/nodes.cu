// Gauss-Legendre nodes and weights, one thread per node, O(1) work per node.
//
// Replaces quadrature.hpp:76-143 (legendre_nodes_weights: Newton on the
// O(N) three-term recurrence, O(N^2) overall). Same contract: theta strictly
// increasing, x = cos(theta) strictly decreasing, w = 2/(dP_N/dtheta)^2, only
// the lower half is solved and the upper half is the exact reflection
// theta_{N-1-k} = pi - theta_k, x_{N-1-k} = -x_k, w_{N-1-k} = w_k
// (quadrature.hpp:126-134); odd N puts (pi/2, 0) in the middle (:135-141).
//
// Newton runs in the perturbation d = theta - theta*_k from the chebstar
// angle theta*_k = (k+3/4) pi / (N+1/2) (the reference's own initial guess,
// quadrature.hpp:84). P_N and dP_N/dtheta come from one of two O(1) formulas:
//
//  * interior (N sin theta >= 25): Stieltjes' expansion
//      P_N(cos t) = C_N sum_m h_m cos((N+m+1/2) t - (m+1/2) pi/2) / (2 sin t)^(m+1/2),
//      h_0 = 1, h_m = h_{m-1} (m-1/2)^2 / (m (N+m+1/2)),
//      C_N = sqrt(4/pi) / ((N+1/2) Lambda(N)),
//    (PAPER.md:262-264 gives the leading term; SURVEY.md 7 H4 the series).
//    Because (N+1/2) theta*_k = (k+3/4) pi exactly, the large phase is reduced
//    symbolically to a quarter-turn index and only (N+1/2) d + m t is
//    rounded, so the node is found to ~1 ulp even at N = 2^26.
//  * boundary (few nodes nearest the endpoints, and all nodes of small N):
//    double-double arithmetic, either the hypergeometric series
//      P_N(cos t) = 2F1(-N, N+1; 1; sin^2(t/2))
//    (N > 128) or the three-term recurrence (N <= 128), so the endpoint
//    nodes do not inherit the eps/sin(theta) error of evaluating P_N at a
//    rounded cos(theta).
#include "common.cuh"
#include "launch.cuh"

namespace flb {

namespace {

// ---- interior: Stieltjes expansion in double ----------------------------
// theta = theta*_k + d; returns P/C_N and (dP/dtheta)/C_N.
__device__ void stieltjes_eval(double n, unsigned long long k, double d, double t, double& P,
                               double& D) {
  double st, ct;
  sincos(t, &st, &ct);
  const double S = 2.0 * st, invS = 1.0 / S, c2 = 2.0 * ct;
  double Sp = rsqrt(S);  // S^-(m+1/2)
  double h = 1.0;
  const double psi0 = (n + 0.5) * d;
  double p = 0.0, dp = 0.0;
  for (int m = 0; m < 48; ++m) {
    if (m > 0) {
      const double mh = (double)m - 0.5;
      h *= mh * mh / ((double)m * (n + (double)m + 0.5));
      Sp *= invS;
      if (h * Sp < 1e-19 * rsqrt(S)) break;
    }
    double sb, cb;
    sincos(psi0 + (double)m * t, &sb, &cb);
    // phase = (pi/2) j + b with j = (2k+1-m) mod 4
    const unsigned q = (unsigned)(((2ull * k + 1ull) + 4ull * 16ull - (unsigned long long)m) & 3ull);
    double cphi, sphi;
    switch (q) {
      case 0: cphi = cb; sphi = sb; break;
      case 1: cphi = -sb; sphi = cb; break;
      case 2: cphi = -cb; sphi = -sb; break;
      default: cphi = sb; sphi = -cb; break;
    }
    const double rho = n + (double)m + 0.5;
    p += h * cphi * Sp;
    dp += h * (-rho * sphi * Sp - ((double)m + 0.5) * cphi * Sp * invS * c2);
  }
  P = p;
  D = dp;
}

// ---- boundary: double-double -------------------------------------------
// P_N(cos t) and dP_N/dt for t in (0, pi/2].
__device__ void boundary_eval(unsigned long long n, dd t, double& P, double& D) {
  const dd half_t = dd_mul_d(t, 0.5);
  const dd sh = dd_sin_small(half_t);                         // sin(t/2)
  const dd s = dd_mul(sh, sh);                                // sin^2(t/2)
  const dd ch = dd_sqrt(dd_sub(dd{1.0, 0.0}, s));             // cos(t/2)
  if (n <= 128) {
    const dd x = dd_sub(dd{1.0, 0.0}, dd_mul_d(s, 2.0));       // cos t
    dd pm1{1.0, 0.0}, p = x;
    for (unsigned long long j = 1; j < n; ++j) {
      const dd a = dd_mul_d(dd_mul(x, p), (double)(2 * j + 1));
      const dd b = dd_mul_d(pm1, (double)j);
      const dd next = dd_div_d(dd_sub(a, b), (double)(j + 1));
      pm1 = p;
      p = next;
    }
    // n == 1: p = x, pm1 = 1
    const dd sint = dd_mul_d(dd_mul(sh, ch), 2.0);
    const dd num = dd_mul_d(dd_sub(dd_mul(x, p), pm1), (double)n);
    P = p.hi;
    D = dd_div(num, sint).hi;
    return;
  }
  // 2F1(-n, n+1; 1; s) = sum_j t_j, t_{j+1} = t_j (j-n)(j+n+1)/(j+1)^2 s
  dd term{1.0, 0.0}, sum{1.0, 0.0}, dsum{0.0, 0.0};
  double tmax = 1.0;
  const double nd = (double)n;
  for (unsigned long long j = 0; j < n && j < 4096; ++j) {
    const double a = (double)j - nd, b = (double)j + nd + 1.0;
    const dd ab = dd_two_prod(a, b);
    const double jp = (double)(j + 1);
    term = dd_mul(dd_div_d(dd_mul(term, ab), jp * jp), s);
    sum = dd_add(sum, term);
    dsum = dd_add(dsum, dd_mul_d(term, jp));
    const double at = fabs(term.hi);
    tmax = fmax(tmax, at);
    if (j > 8 && at < 1e-40 * tmax) break;
  }
  P = sum.hi;
  // dP/dt = (sum_j j t_j) * cos(t/2) / sin(t/2)
  D = dd_div(dd_mul(dsum, ch), sh).hi;
}

// theta*_k as a double-double: (k + 3/4) pi / (n + 1/2)
__device__ dd theta_star_dd(unsigned long long n, unsigned long long k) {
  const dd pi{kPiHi, kPiLo};
  return dd_div_d(dd_mul_d(pi, (double)k + 0.75), (double)n + 0.5);
}

__global__ void nodes_kernel(unsigned long long n, double* __restrict__ theta,
                             double* __restrict__ xo, double* __restrict__ wo, double cn) {
  const unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long half = n / 2;
  const bool odd = (n & 1ull) != 0;
  if (k > half || (k == half && !odd)) return;
  const double nd = (double)n;
  const dd tstar = theta_star_dd(n, k);
  const bool mid = odd && k == half;  // theta*_mid = pi/2 exactly
  const bool interior = nd * sin(tstar.hi) >= 25.0;

  double d = 0.0, P = 0.0, D = 1.0;
  if (!mid) {
    for (int it = 0; it < 12; ++it) {
      if (interior) {
        stieltjes_eval(nd, k, d, tstar.hi + d, P, D);
      } else {
        boundary_eval(n, dd_add_d(tstar, d), P, D);
      }
      const double step = P / D;
      d -= step;
      if (fabs(step) <= 1e-20 * tstar.hi) break;
    }
  }
  // derivative at the converged angle, for the weight
  double th;
  if (mid) {
    th = 0.5 * kPi;
  } else {
    const dd tt = dd_add_d(tstar, d);
    th = tt.hi;  // round to double: fl(theta*_k + d)
  }
  double w;
  if (interior) {
    stieltjes_eval(nd, k, d, tstar.hi + d, P, D);
    const double dpt = cn * D;
    w = 2.0 / (dpt * dpt);
  } else {
    boundary_eval(n, mid ? dd{kPiHi * 0.5, kPiLo * 0.5} : dd_add_d(tstar, d), P, D);
    w = 2.0 / (D * D);
  }
  // x = cos(theta) of the rounded theta, in double-double: 1 - 2 sin^2(theta/2)
  double x;
  if (mid) {
    x = 0.0;
  } else {
    const dd sh = dd_sin_small(dd{th * 0.5, 0.0});
    x = dd_sub(dd{1.0, 0.0}, dd_mul_d(dd_mul(sh, sh), 2.0)).hi;
  }
  theta[k] = th;
  xo[k] = x;
  wo[k] = w;
  if (!mid) {
    theta[n - 1 - k] = __dsub_rn(kPi, th);  // quadrature.hpp:131
    xo[n - 1 - k] = -x;
    wo[n - 1 - k] = w;
  }
}

// quadrature.hpp:32-36 + :147-158, same operation order, no contraction
__global__ void reference_grid_kernel(unsigned long long n, int kind,
                                      const double* __restrict__ theta,
                                      double* __restrict__ theta_star,
                                      double* __restrict__ delta) {
  const unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double ts;
  if (kind == FL_CHEB1)
    ts = __ddiv_rn(__dmul_rn(__dadd_rn((double)k, 0.5), kPi), (double)n);
  else
    ts = __ddiv_rn(__dmul_rn(__dadd_rn((double)k, 0.75), kPi), __dadd_rn((double)n, 0.5));
  if (theta_star) theta_star[k] = ts;
  if (delta) delta[k] = __dsub_rn(theta[k], ts);
}

// conversion.hpp:43-56 (asymptotic sqrt(z) Lambda(z), < 1 ulp for z >= 30)
__host__ __device__ inline double lambda_asymptotic(double z) {
  const double k1 = -1.0 / 8.0, k2 = 1.0 / 128.0, k3 = 5.0 / 1024.0, k4 = -21.0 / 32768.0;
  const double k5 = -399.0 / 262144.0, k6 = 869.0 / 4194304.0, k7 = 39325.0 / 33554432.0;
  const double k8 = -334477.0 / 2147483648.0;
  const double r = 1.0 / z;
  const double s =
      1.0 + r * (k1 + r * (k2 + r * (k3 + r * (k4 + r * (k5 + r * (k6 + r * (k7 + r * k8)))))));
  return s / sqrt(z);
}

// Lambda(z) = Gamma(z+1/2)/Gamma(z+1) for z <= max_index: the reference's
// recurrence (conversion.hpp:25-30) for z < 64 (one thread, same rounding
// chain), the sub-ulp asymptotic series above that, one thread per entry.
__global__ void lambda_kernel(unsigned long long max_index, double* __restrict__ table) {
  const unsigned long long z = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (z > max_index) return;
  if (z == 0) {
    double v = sqrt(kPi);
    table[0] = v;
    for (unsigned long long i = 0; i + 1 <= max_index && i + 1 < 64; ++i) {
      v = v * ((double)i + 0.5) / ((double)i + 1.0);
      table[i + 1] = v;
    }
    return;
  }
  if (z < 64) return;
  table[z] = lambda_asymptotic((double)z);
}

}  // namespace

double lambda_value_host(unsigned long long z) {
  if (z >= 30) return lambda_asymptotic((double)z);
  double v = sqrt(kPi);
  for (unsigned long long i = 0; i < z; ++i) v = v * ((double)i + 0.5) / ((double)i + 1.0);
  return v;
}

void launch_nodes(size_t n, double* theta, double* x, double* w, cudaStream_t s) {
  const size_t count = n / 2 + 1;
  // C_N = sqrt(4/pi) / ((N+1/2) Lambda(N))
  const double cn = sqrt(4.0 / kPi) / (((double)n + 0.5) * lambda_value_host(n));
  const int threads = 128;
  nodes_kernel<<<(unsigned)((count + threads - 1) / threads), threads, 0, s>>>(n, theta, x, w, cn);
  note_launch("nodes_kernel");
}

void launch_reference_grid(size_t n, int kind, const double* theta, double* theta_star,
                           double* delta, cudaStream_t s) {
  const int threads = 256;
  reference_grid_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(
      n, kind, theta, theta_star, delta);
  note_launch("reference_grid_kernel");
}

void launch_lambda(size_t max_index, double* table, cudaStream_t s) {
  const int threads = 256;
  const size_t count = max_index + 1;
  lambda_kernel<<<(unsigned)((count + threads - 1) / threads), threads, 0, s>>>(max_index, table);
  note_launch("lambda_kernel");
}

}  // namespace flb
