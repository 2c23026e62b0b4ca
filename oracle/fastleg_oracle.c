/* TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference hot path.
 * See fastleg_oracle.h for the contract. Citations are to
 * /root/reference/proj/include/fastleg/<file>:<line>.
 *
 * Compiled with -ffp-contract=off so that the operation order written here
 * is the rounding order (the reference is restated expression by
 * expression, so the two agree bit-for-bit when built with the same flags).
 */
#include "fastleg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "r2r.h"

/* types.hpp:36 */
static const double FO_PI = 3.14159265358979323846264338327950288;

/* quadrature.hpp:32-36 reference_angle */
double fo_reference_angle(size_t n, int kind, size_t k) {
  if (kind == FO_CHEB1) return ((double)k + 0.5) * FO_PI / (double)n;
  return ((double)k + 0.75) * FO_PI / ((double)n + 0.5);
}

/* quadrature.hpp:43-57 detail::legendre_pair_batch */
static void legendre_pair_batch(size_t n, const double* x, size_t m, double* p_n,
                                double* p_nm1) {
  for (size_t k = 0; k < m; ++k) {
    p_nm1[k] = 1.0;
    p_n[k] = x[k];
  }
  for (size_t j = 1; j < n; ++j) {
    const double a = (2.0 * (double)j + 1.0) / ((double)j + 1.0);
    const double b = (double)j / ((double)j + 1.0);
    for (size_t k = 0; k < m; ++k) {
      const double next = a * x[k] * p_n[k] - b * p_nm1[k];
      p_nm1[k] = p_n[k];
      p_n[k] = next;
    }
  }
}

/* quadrature.hpp:60-68 detail::legendre_prev_at_zero */
static double legendre_prev_at_zero(size_t n) {
  double p_prev = 1.0, p = 0.0;
  for (size_t j = 1; j + 1 < n; ++j) {
    const double next = -(double)j * p_prev / ((double)j + 1.0);
    p_prev = p;
    p = next;
  }
  return n >= 2 ? p : p_prev;
}

/* quadrature.hpp:76-143 legendre_nodes_weights (Newton in theta from the
 * chebstar angles, lower half only, reflection for the rest) */
int fo_legendre_nodes_weights(size_t n, double* theta, double* xout, double* wout) {
  if (n == 0) return 1; /* :77 invalid_argument */
  const size_t half = n / 2;
  double* th = (double*)malloc(sizeof(double) * (half + 1));
  double* x = (double*)malloc(sizeof(double) * (half + 1));
  double* p_n = (double*)malloc(sizeof(double) * (half + 1));
  double* p_nm1 = (double*)malloc(sizeof(double) * (half + 1));
  double* dpdth = (double*)malloc(sizeof(double) * (half + 1));
  double* prev_step = (double*)malloc(sizeof(double) * (half + 1));
  char* active = (char*)malloc(half + 1);
  for (size_t k = 0; k < half; ++k) {
    th[k] = fo_reference_angle(n, FO_CHEBSTAR, k);
    prev_step[k] = INFINITY;
    active[k] = 1;
  }
  const double step_tol = 1e-15, noise_ceiling = 1e-11; /* :91-93 */
  const int max_iterations = 12;
  size_t remaining = half;
  for (int it = 0; it < max_iterations && remaining > 0; ++it) { /* :96-111 */
    for (size_t k = 0; k < half; ++k) x[k] = cos(th[k]);
    legendre_pair_batch(n, x, half, p_n, p_nm1);
    for (size_t k = 0; k < half; ++k) {
      if (!active[k]) continue;
      const double dp = (double)n * (x[k] * p_n[k] - p_nm1[k]) / sin(th[k]);
      const double step = p_n[k] / dp;
      th[k] -= step;
      const double mag = fabs(step);
      if (mag <= step_tol || (mag <= noise_ceiling && mag >= 0.01 * prev_step[k])) {
        active[k] = 0;
        --remaining;
      }
      prev_step[k] = mag;
    }
  }
  int status = 0;
  if (remaining > 0) {
    status = 4; /* :112-113 runtime_error */
  } else {
    for (size_t k = 0; k < half; ++k) x[k] = cos(th[k]); /* :116-119 */
    legendre_pair_batch(n, x, half, p_n, p_nm1);
    for (size_t k = 0; k < half; ++k)
      dpdth[k] = (double)n * (x[k] * p_n[k] - p_nm1[k]) / sin(th[k]);
    for (size_t k = 0; k < half; ++k) { /* :126-134 */
      const double w = 2.0 / (dpdth[k] * dpdth[k]);
      theta[k] = th[k];
      theta[n - 1 - k] = FO_PI - th[k];
      xout[k] = x[k];
      xout[n - 1 - k] = -x[k];
      wout[k] = w;
      wout[n - 1 - k] = w;
    }
    if (n % 2 == 1) { /* :135-141 */
      const size_t mid = (n - 1) / 2;
      const double dp_mid = (double)n * legendre_prev_at_zero(n);
      theta[mid] = 0.5 * FO_PI;
      xout[mid] = 0.0;
      wout[mid] = 2.0 / (dp_mid * dp_mid);
    }
  }
  free(th); free(x); free(p_n); free(p_nm1); free(dpdth); free(prev_step); free(active);
  return status;
}

/* quadrature.hpp:147-158 reference_grid */
int fo_reference_grid(size_t n, int kind, const double* theta, double* theta_star,
                      double* delta) {
  for (size_t k = 0; k < n; ++k) {
    theta_star[k] = fo_reference_angle(n, kind, k);
    delta[k] = theta[k] - theta_star[k];
  }
  return 0;
}

/* ---------------- trig.hpp ---------------- */

/* trig.hpp:55-74 dct_iii */
int fo_dct_iii(size_t n, int kind, const double* c, double* out) {
  if (n == 0) return 1; /* :50 */
  if (kind == FO_CHEB1) {
    double* in = (double*)malloc(sizeof(double) * n);
    in[0] = c[0];
    for (size_t j = 1; j < n; ++j) in[j] = 0.5 * c[j];
    int rc = r2r_execute(R2R_REDFT01, n, in, out);
    free(in);
    return rc ? 4 : 0;
  }
  const size_t m = 2 * n + 1;
  double* in = (double*)calloc(m, sizeof(double));
  double* o = (double*)malloc(sizeof(double) * m);
  in[0] = c[0];
  for (size_t j = 1; j < n; ++j) in[j] = 0.5 * c[j];
  int rc = r2r_execute(R2R_REDFT01, m, in, o);
  for (size_t k = 0; k < n; ++k) out[k] = o[2 * k + 1];
  free(in);
  free(o);
  return rc ? 4 : 0;
}

/* trig.hpp:76-95 dst_iii */
int fo_dst_iii(size_t n, int kind, const double* c, double* out) {
  if (n == 0) return 1;
  if (kind == FO_CHEB1) {
    if (n == 1) {
      out[0] = 0.0;
      return 0;
    }
    double* in = (double*)calloc(n, sizeof(double));
    for (size_t j = 0; j + 1 < n; ++j) in[j] = 0.5 * c[j + 1];
    int rc = r2r_execute(R2R_RODFT01, n, in, out);
    free(in);
    return rc ? 4 : 0;
  }
  const size_t m = 2 * n + 1;
  double* in = (double*)calloc(m, sizeof(double));
  double* o = (double*)malloc(sizeof(double) * m);
  for (size_t j = 0; j + 1 < n; ++j) in[j] = 0.5 * c[j + 1];
  int rc = r2r_execute(R2R_RODFT01, m, in, o);
  for (size_t k = 0; k < n; ++k) out[k] = o[2 * k + 1];
  free(in);
  free(o);
  return rc ? 4 : 0;
}

/* trig.hpp:100-116 dct_iii_transpose */
int fo_dct_iii_transpose(size_t n, int kind, const double* g, double* out) {
  if (n == 0) return 1;
  if (kind == FO_CHEB1) {
    int rc = r2r_execute(R2R_REDFT10, n, g, out);
    for (size_t j = 0; j < n; ++j) out[j] *= 0.5;
    return rc ? 4 : 0;
  }
  const size_t m = 2 * n + 1;
  double* in = (double*)calloc(m, sizeof(double));
  double* o = (double*)malloc(sizeof(double) * m);
  for (size_t k = 0; k < n; ++k) in[2 * k + 1] = g[k];
  int rc = r2r_execute(R2R_REDFT10, m, in, o);
  for (size_t j = 0; j < n; ++j) out[j] = 0.5 * o[j];
  free(in);
  free(o);
  return rc ? 4 : 0;
}

/* trig.hpp:118-136 dst_iii_transpose */
int fo_dst_iii_transpose(size_t n, int kind, const double* g, double* out) {
  if (n == 0) return 1;
  for (size_t j = 0; j < n; ++j) out[j] = 0.0;
  if (kind == FO_CHEB1) {
    if (n == 1) return 0;
    double* o = (double*)malloc(sizeof(double) * n);
    int rc = r2r_execute(R2R_RODFT10, n, g, o);
    for (size_t j = 1; j < n; ++j) out[j] = 0.5 * o[j - 1];
    free(o);
    return rc ? 4 : 0;
  }
  const size_t m = 2 * n + 1;
  double* in = (double*)calloc(m, sizeof(double));
  double* o = (double*)malloc(sizeof(double) * m);
  for (size_t k = 0; k < n; ++k) in[2 * k + 1] = g[k];
  int rc = r2r_execute(R2R_RODFT10, m, in, o);
  for (size_t j = 1; j < n; ++j) out[j] = 0.5 * o[j - 1];
  free(in);
  free(o);
  return rc ? 4 : 0;
}

/* ---------------- ndct.hpp ---------------- */

/* ndct.hpp:38-44 taylor_term_bound (negative counts: caller's check) */
double fo_taylor_term_bound(int kind, int num_terms) {
  const double q = kind == FO_CHEB1 ? 0.83845 : 1.0 / (6.0 * FO_PI);
  double bound = 1.0;
  for (int l = 1; l <= num_terms; ++l) bound *= q / (double)l;
  return bound;
}

/* ndct.hpp:49-59 min_taylor_terms (max_taylor_terms = 30, :46) */
int fo_min_taylor_terms(int kind, double tolerance, int* terms) {
  if (!(tolerance > 0.0 && tolerance < 1.0)) return 1;
  const double q = kind == FO_CHEB1 ? 0.83845 : 1.0 / (6.0 * FO_PI);
  double bound = 1.0;
  for (int l = 1; l <= 30; ++l) {
    bound *= q / (double)l;
    if (bound <= tolerance) {
      *terms = l;
      return 0;
    }
  }
  return 2;
}

/* ndct.hpp:77 */
static int taylor_sign(int l) { return ((l + 1) / 2) % 2 == 0 ? 1 : -1; }

/* ndct.hpp:79-91 check_ndct_input (size checked by the caller) */
static int check_ndct_input(size_t n, int num_terms, const double* v) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 1;
  if (n > 1 && (double)(num_terms - 1) * log10((double)(n - 1)) > 300.0) return 3;
  return 0;
}

typedef int (*trig_fn)(size_t, int, const double*, double*);

/* ndct.hpp:98-117 ndct_apply */
int fo_ndct_apply(size_t n, int kind, int num_terms, const double* delta, const double* c,
                  double* f) {
  int rc = check_ndct_input(n, num_terms, c);
  if (rc) return rc;
  double* stage = (double*)malloc(sizeof(double) * n);
  double* perturb_pow = (double*)malloc(sizeof(double) * n);
  double* t = (double*)malloc(sizeof(double) * n);
  for (size_t j = 0; j < n; ++j) {
    f[j] = 0.0;
    stage[j] = c[j];
    perturb_pow[j] = 1.0;
  }
  for (int l = 0; l < num_terms && rc == 0; ++l) {
    if (l > 0) {
      for (size_t j = 0; j < n; ++j) {
        stage[j] *= (double)j;
        perturb_pow[j] *= delta[j] / (double)l;
      }
    }
    rc = (l % 2 == 0 ? fo_dct_iii : fo_dst_iii)(n, kind, stage, t);
    const double sign = (double)taylor_sign(l);
    for (size_t k = 0; k < n; ++k) f[k] += sign * perturb_pow[k] * t[k];
  }
  free(stage);
  free(perturb_pow);
  free(t);
  return rc;
}

/* ndct.hpp:121-143 ndct_apply_transpose */
int fo_ndct_apply_transpose(size_t n, int kind, int num_terms, const double* delta,
                            const double* g, double* out) {
  int rc = check_ndct_input(n, num_terms, g);
  if (rc) return rc;
  double* degree_pow = (double*)malloc(sizeof(double) * n);
  double* perturb_pow = (double*)malloc(sizeof(double) * n);
  double* h = (double*)malloc(sizeof(double) * n);
  double* t = (double*)malloc(sizeof(double) * n);
  for (size_t j = 0; j < n; ++j) {
    out[j] = 0.0;
    degree_pow[j] = 1.0;
    perturb_pow[j] = 1.0;
  }
  for (int l = 0; l < num_terms && rc == 0; ++l) {
    if (l > 0) {
      for (size_t j = 0; j < n; ++j) {
        degree_pow[j] *= (double)j;
        perturb_pow[j] *= delta[j] / (double)l;
      }
    }
    for (size_t k = 0; k < n; ++k) h[k] = perturb_pow[k] * g[k];
    rc = (l % 2 == 0 ? fo_dct_iii_transpose : fo_dst_iii_transpose)(n, kind, h, t);
    const double sign = (double)taylor_sign(l);
    for (size_t j = 0; j < n; ++j) out[j] += sign * degree_pow[j] * t[j];
  }
  free(degree_pow);
  free(perturb_pow);
  free(h);
  free(t);
  return rc;
}

/* ndct.hpp:147-155 ndct_error_bound */
double fo_ndct_error_bound(size_t n, int kind, int num_terms, const double* delta,
                           const double* c) {
  double max_perturb = 0.0;
  for (size_t k = 0; k < n; ++k) {
    const double d = fabs(delta[k]);
    if (max_perturb < d) max_perturb = d;
  }
  const double q = (double)n * max_perturb;
  double node_bound = 1.0;
  for (int l = 1; l <= num_terms; ++l) node_bound *= q / (double)l;
  const double grid_bound = fo_taylor_term_bound(kind, num_terms);
  double s = 0.0; /* types.hpp:38-42 norm_l1 */
  for (size_t k = 0; k < n; ++k) s += c[k] < 0 ? -c[k] : c[k];
  return (grid_bound < node_bound ? grid_bound : node_bound) * s;
}

/* ---------------- conversion.hpp ---------------- */

/* conversion.hpp:25-30 LambdaCache */
void fo_lambda_table(size_t max_index, double* table) {
  table[0] = sqrt(FO_PI);
  for (size_t z = 0; z + 1 <= max_index; ++z)
    table[z + 1] = table[z] * ((double)z + 0.5) / ((double)z + 1.0);
}

/* conversion.hpp:43-56 lambda_ratio_asymptotic */
static double lambda_ratio_asymptotic(double z) {
  const double k1 = -1.0 / 8.0, k2 = 1.0 / 128.0, k3 = 5.0 / 1024.0, k4 = -21.0 / 32768.0;
  const double k5 = -399.0 / 262144.0, k6 = 869.0 / 4194304.0, k7 = 39325.0 / 33554432.0;
  const double k8 = -334477.0 / 2147483648.0;
  const double r = 1.0 / z;
  const double s =
      1.0 + r * (k1 + r * (k2 + r * (k3 + r * (k4 + r * (k5 + r * (k6 + r * (k7 + r * k8)))))));
  return s / sqrt(z);
}

/* conversion.hpp:63-73 lambda_ratio */
int fo_lambda_ratio(double z, const double* table, size_t max_index, double* out) {
  if (!(z >= 0.0)) return 2;
  const double zf = floor(z);
  if (z == zf && zf <= (double)max_index) {
    *out = table[(size_t)zf];
    return 0;
  }
  if (z >= 30.0) {
    *out = lambda_ratio_asymptotic(z);
    return 0;
  }
  const double frac = z - zf;
  double value = exp(lgamma(frac + 0.5) - lgamma(frac + 1.0));
  for (double w = frac; w < z - 0.5; w += 1.0) value *= (w + 0.5) / (w + 1.0);
  *out = value;
  return 0;
}

/* conversion.hpp:76-81 leg2cheb_entry */
double fo_leg2cheb_entry(size_t k, size_t n, const double* table, size_t max_index) {
  if (k > n || (k + n) % 2 != 0) return 0.0;
  const double prefactor = (k == 0 ? 1.0 : 2.0) / FO_PI;
  double a = 0, b = 0;
  fo_lambda_ratio((double)((n - k) / 2), table, max_index, &a);
  fo_lambda_ratio((double)((n + k) / 2), table, max_index, &b);
  return prefactor * a * b;
}

/* conversion.hpp:88-94 scaled_lambda_table */
static int scaled_lambda_table(const double* table, size_t max_index, size_t count, double* s) {
  if (count > 0 && max_index + 1 < count) return 1;
  for (size_t j = 0; j < count; ++j) s[j] = table[j] / table[0];
  return 0;
}

/* conversion.hpp:100-113 leg2cheb_apply (basis check is the caller's) */
int fo_leg2cheb_apply(size_t n, const double* table, size_t max_index, const double* c,
                      double* out) {
  double* s = (double*)malloc(sizeof(double) * (n + 1));
  int rc = scaled_lambda_table(table, max_index, n, s);
  if (rc == 0) {
    /* rows are independent and each keeps the reference's summation order, so
       the row-parallel loop is bit-identical to the serial one (OpenMP only
       shortens the O(N^2) oracle at N >= 2^16) */
#pragma omp parallel for schedule(dynamic, 64) if (n >= 4096)
    for (size_t k = 0; k < n; ++k) {
      double acc = 0.0;
      for (size_t j = 0; k + 2 * j < n; ++j) acc += s[j] * s[k + j] * c[k + 2 * j];
      out[k] = (k == 0 ? 1.0 : 2.0) * acc;
    }
  }
  free(s);
  return rc;
}

/* conversion.hpp:121-135 leg2cheb_apply_transpose */
int fo_leg2cheb_apply_transpose(size_t n, const double* table, size_t max_index,
                                const double* v, double* out) {
  double* s = (double*)malloc(sizeof(double) * (n + 1));
  int rc = scaled_lambda_table(table, max_index, n, s);
  if (rc == 0) {
#pragma omp parallel for schedule(dynamic, 64) if (n >= 4096)
    for (size_t m = 0; m < n; ++m) {
      double acc = 0.0;
      for (size_t j = 0; 2 * j < m; ++j) acc += s[j] * s[m - j] * v[m - 2 * j];
      acc *= 2.0;
      if (m % 2 == 0) acc += s[m / 2] * s[m - m / 2] * v[0];
      out[m] = acc;
    }
  }
  free(s);
  return rc;
}

/* ---------------- transforms.hpp (grid injected) ---------------- */

/* transforms.hpp:42-49 dlt = ndct_apply(plan, leg2cheb_apply(c, lambda)) */
int fo_dlt_grid(size_t n, int kind, int num_terms, const double* delta, const double* c,
                double* f) {
  double* table = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* cheb = (double*)malloc(sizeof(double) * (n ? n : 1));
  fo_lambda_table(n - 1, table); /* transforms.hpp:24 lambda_(n - 1) */
  int rc = fo_leg2cheb_apply(n, table, n - 1, c, cheb);
  if (rc == 0) rc = fo_ndct_apply(n, kind, num_terms, delta, cheb, f);
  free(table);
  free(cheb);
  return rc;
}

/* transforms.hpp:54-64 idlt */
int fo_idlt_grid(size_t n, int kind, int num_terms, const double* delta, const double* weights,
                 const double* f, double* c) {
  double* table = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* weighted = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* back = (double*)malloc(sizeof(double) * (n ? n : 1));
  fo_lambda_table(n - 1, table);
  for (size_t k = 0; k < n; ++k) weighted[k] = weights[k] * f[k];
  int rc = fo_ndct_apply_transpose(n, kind, num_terms, delta, weighted, back);
  if (rc == 0) rc = fo_leg2cheb_apply_transpose(n, table, n - 1, back, c);
  if (rc == 0)
    for (size_t m = 0; m < n; ++m) c[m] *= (double)m + 0.5;
  free(table);
  free(weighted);
  free(back);
  return rc;
}

/* ---------------- oracle.hpp ---------------- */

/* oracle.hpp:19-48 eval_legendre_direct */
int fo_eval_legendre_direct(size_t n, const double* c, size_t m, const double* xs, double* out) {
  for (size_t j = 0; j < m; ++j)
    if (!(fabs(xs[j]) <= 1.0)) return 2;
  for (size_t j = 0; j < m; ++j) {
    const double x = xs[j];
    double p_prev = 1.0;
    double acc = n > 0 ? c[0] : 0.0;
    if (n > 1) {
      double p = x;
      acc += c[1] * p;
      for (size_t q = 1; q + 1 < n; ++q) {
        const double next = ((2.0 * (double)q + 1.0) * x * p - (double)q * p_prev) / ((double)q + 1.0);
        p_prev = p;
        p = next;
        acc += c[q + 1] * p;
      }
    }
    out[j] = acc;
  }
  return 0;
}

/* oracle.hpp:52-79 eval_chebyshev_direct */
int fo_eval_chebyshev_direct(size_t n, const double* c, size_t m, const double* xs, double* out) {
  for (size_t j = 0; j < m; ++j)
    if (!(fabs(xs[j]) <= 1.0)) return 2;
  for (size_t j = 0; j < m; ++j) {
    const double x = xs[j];
    double t_prev = 1.0;
    double acc = n > 0 ? c[0] : 0.0;
    if (n > 1) {
      double t = x;
      acc += c[1] * t;
      for (size_t q = 1; q + 1 < n; ++q) {
        const double next = 2.0 * x * t - t_prev;
        t_prev = t;
        t = next;
        acc += c[q + 1] * next;
      }
    }
    out[j] = acc;
  }
  return 0;
}

/* oracle.hpp:84-116 idlt_direct */
int fo_idlt_direct(size_t n, const double* f, const double* x, const double* w, double* out) {
  double* wf = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* p_prev = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* p = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (size_t k = 0; k < n; ++k) {
    wf[k] = w[k] * f[k];
    p_prev[k] = 1.0;
    out[k] = 0.0;
  }
  double acc = 0.0;
  for (size_t k = 0; k < n; ++k) acc += wf[k];
  if (n > 0) out[0] = 0.5 * acc;
  if (n > 1) {
    for (size_t k = 0; k < n; ++k) p[k] = x[k];
    acc = 0.0;
    for (size_t k = 0; k < n; ++k) acc += wf[k] * p[k];
    out[1] = 1.5 * acc;
    for (size_t m = 1; m + 1 < n; ++m) {
      const double a = (2.0 * (double)m + 1.0) / ((double)m + 1.0);
      const double b = (double)m / ((double)m + 1.0);
      acc = 0.0;
      for (size_t k = 0; k < n; ++k) {
        const double next = a * x[k] * p[k] - b * p_prev[k];
        p_prev[k] = p[k];
        p[k] = next;
        acc += wf[k] * next;
      }
      out[m + 1] = ((double)(m + 1) + 0.5) * acc;
    }
  }
  free(wf);
  free(p_prev);
  free(p);
  return 0;
}

/* oracle.hpp:122-153 cheb_coeffs_of_legendre; out has n+1 entries */
int fo_cheb_coeffs_of_legendre(size_t n, size_t m, double* out) {
  if (m <= n) return 1;
  double* samples = (double*)malloc(sizeof(double) * m);
  for (size_t j = 0; j < m; ++j) {
    const double x = cos(((double)j + 0.5) * FO_PI / (double)m);
    double p_prev = 1.0, p = x;
    if (n == 0) {
      samples[j] = 1.0;
      continue;
    }
    for (size_t q = 1; q < n; ++q) {
      const double next = ((2.0 * (double)q + 1.0) * x * p - (double)q * p_prev) / ((double)q + 1.0);
      p_prev = p;
      p = next;
    }
    samples[j] = p;
  }
  for (size_t k = 0; k <= n; ++k) {
    double acc = 0.0;
    for (size_t j = 0; j < m; ++j)
      acc += samples[j] * cos((double)k * ((double)j + 0.5) * FO_PI / (double)m);
    out[k] = (k == 0 ? 1.0 : 2.0) / (double)m * acc;
  }
  free(samples);
  return 0;
}

/* ---------------- random.hpp ---------------- */

/* std::mt19937_64 (the 64-bit Mersenne Twister the C++ standard pins). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  if (s->idx >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (s->mt[i] & upper) | (s->mt[(i + 1) % 312] & lower);
      uint64_t v = s->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = v;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

uint64_t fo_mt19937_64_nth(uint64_t seed, uint64_t count) {
  mt64 s;
  mt64_seed(&s, seed);
  uint64_t v = 0;
  for (uint64_t i = 0; i < count; ++i) v = mt64_next(&s);
  return v;
}

/* random.hpp:36 uniform01 */
static double uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }

/* random.hpp:15-41 GaussianSource::next + :45-55 random_decaying */
void fo_random_decaying(size_t n, double decay, uint64_t seed, double* out) {
  mt64 s;
  mt64_seed(&s, seed);
  int have_spare = 0;
  double spare = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double g;
    if (have_spare) {
      have_spare = 0;
      g = spare;
    } else {
      double u1 = 0.0;
      do {
        u1 = uniform01(&s);
      } while (u1 == 0.0);
      const double u2 = uniform01(&s);
      const double r = sqrt(-2.0 * log(u1));
      have_spare = 1;
      spare = r * sin(2.0 * FO_PI * u2);
      g = r * cos(2.0 * FO_PI * u2);
    }
    out[i] = g * pow((double)(i + 1), -decay);
  }
}

/* SURVEY.md 8d C4 recipe: u = 2 * uniform01 - 1 from mt19937_64(seed) */
void fo_uniform_pm1(size_t n, uint64_t seed, double* out) {
  mt64 s;
  mt64_seed(&s, seed);
  for (size_t i = 0; i < n; ++i) out[i] = 2.0 * uniform01(&s) - 1.0;
}
