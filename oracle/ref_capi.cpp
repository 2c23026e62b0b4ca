// TEST INFRASTRUCTURE ONLY -- C wrappers over the UNMODIFIED reference headers
// (/root/reference/proj/include/fastleg/*.hpp), compiled in place by
// oracle/Makefile against the FFTW-API shim (oracle/fftw_shim/fftw3.h) into
// oracle/_ref/libfastleg_ref.so. Used by tests/ to pin the C restatement and
// the GPU path, and by bench.py --impl reference as the CPU baseline.
// Return codes as in fastleg_oracle.h.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "fastleg/fastleg.hpp"

using namespace fastleg;

namespace {

GridKind kind_of(int k) { return k == 0 ? GridKind::cheb1 : GridKind::chebstar; }

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::domain_error&) {
    return 2;
  } catch (const std::overflow_error&) {
    return 3;
  } catch (const std::runtime_error&) {
    return 4;
  } catch (...) {
    return 5;
  }
}

std::vector<double> vec(const double* p, std::size_t n) { return std::vector<double>(p, p + n); }
void put(const std::vector<double>& v, double* out) { std::memcpy(out, v.data(), v.size() * 8); }

TaylorPlan make_plan(std::size_t n, int kind, int num_terms, const double* delta) {
  TaylorPlan plan;
  plan.size = n;
  plan.kind = kind_of(kind);
  plan.tolerance = default_tolerance;
  plan.num_terms = num_terms;
  plan.reference.size = n;
  plan.reference.kind = plan.kind;
  plan.reference.delta_theta = vec(delta, n);
  plan.reference.theta_star.resize(n);
  for (std::size_t k = 0; k < n; ++k) plan.reference.theta_star[k] = reference_angle(n, plan.kind, k);
  return plan;
}

}  // namespace

extern "C" {

int fr_legendre_nodes_weights(std::size_t n, double* theta, double* x, double* w) {
  return guard([&] {
    const LegendreGrid g = legendre_nodes_weights(n);
    put(g.theta, theta);
    put(g.x, x);
    put(g.weights, w);
  });
}

int fr_reference_grid(std::size_t n, int kind, const double* theta, double* theta_star,
                      double* delta) {
  return guard([&] {
    LegendreGrid g;
    g.size = n;
    g.theta = vec(theta, n);
    const ReferenceGrid r = reference_grid(g, kind_of(kind));
    put(r.theta_star, theta_star);
    put(r.delta_theta, delta);
  });
}

int fr_trig(int op, std::size_t n, int kind, const double* in, double* out) {
  return guard([&] {
    const std::vector<double> v = vec(in, n);
    std::vector<double> r;
    switch (op) {
      case 0: r = dct_iii(v, kind_of(kind)); break;
      case 1: r = dst_iii(v, kind_of(kind)); break;
      case 2: r = dct_iii_transpose(v, kind_of(kind)); break;
      default: r = dst_iii_transpose(v, kind_of(kind)); break;
    }
    put(r, out);
  });
}

int fr_min_taylor_terms(int kind, double tol, int* terms) {
  return guard([&] { *terms = min_taylor_terms(kind_of(kind), tol); });
}

double fr_taylor_term_bound(int kind, int num_terms) {
  return taylor_term_bound(kind_of(kind), num_terms);
}

int fr_ndct(int transpose, std::size_t n, int kind, int num_terms, const double* delta,
            const double* in, double* out) {
  return guard([&] {
    const TaylorPlan plan = make_plan(n, kind, num_terms, delta);
    const std::vector<double> v = vec(in, n);
    put(transpose ? ndct_apply_transpose(plan, v) : ndct_apply(plan, v), out);
  });
}

double fr_ndct_error_bound(std::size_t n, int kind, int num_terms, const double* delta,
                           const double* c) {
  const TaylorPlan plan = make_plan(n, kind, num_terms, delta);
  return ndct_error_bound(plan, vec(c, n));
}

int fr_lambda_table(std::size_t max_index, double* table) {
  return guard([&] {
    const LambdaCache cache(max_index);
    for (std::size_t z = 0; z <= max_index; ++z) table[z] = cache[z];
  });
}

int fr_lambda_ratio(double z, std::size_t max_index, double* out) {
  return guard([&] {
    const LambdaCache cache(max_index);
    *out = lambda_ratio(z, cache);
  });
}

double fr_leg2cheb_entry(std::size_t k, std::size_t n, std::size_t max_index) {
  const LambdaCache cache(max_index);
  return leg2cheb_entry(k, n, cache);
}

int fr_leg2cheb(int transpose, std::size_t n, const double* in, double* out) {
  return guard([&] {
    const LambdaCache cache(n == 0 ? 0 : n - 1);
    if (transpose)
      put(leg2cheb_apply_transpose(vec(in, n), cache), out);
    else
      put(leg2cheb_apply(legendre_coefficients(vec(in, n)), cache).values, out);
  });
}

// transforms.hpp:42-64 with an injected grid (theta, x, weights)
int fr_dlt_grid(std::size_t n, int kind, double tol, const double* theta, const double* x,
                const double* w, const double* c, double* f) {
  return guard([&] {
    LegendreGrid g{n, vec(theta, n), vec(x, n), vec(w, n)};
    const TaylorPlan plan = plan_ndct(g, kind_of(kind), tol);
    const LambdaCache cache(n - 1);
    const CoefficientVector cheb = leg2cheb_apply(legendre_coefficients(vec(c, n)), cache);
    put(ndct_apply(plan, cheb.values), f);
  });
}

int fr_idlt_grid(std::size_t n, int kind, double tol, const double* theta, const double* x,
                 const double* w, const double* f, double* c) {
  return guard([&] {
    LegendreGrid g{n, vec(theta, n), vec(x, n), vec(w, n)};
    const TaylorPlan plan = plan_ndct(g, kind_of(kind), tol);
    const LambdaCache cache(n - 1);
    std::vector<double> weighted(n);
    for (std::size_t k = 0; k < n; ++k) weighted[k] = g.weights[k] * f[k];
    const std::vector<double> back = ndct_apply_transpose(plan, weighted);
    std::vector<double> coeffs = leg2cheb_apply_transpose(back, cache);
    for (std::size_t m = 0; m < n; ++m) coeffs[m] *= static_cast<double>(m) + 0.5;
    put(coeffs, c);
  });
}

// The stock composed API (TransformConfig builds its own Newton grid).
struct fr_config {
  TransformConfig cfg;
  fr_config(std::size_t n, double tol, GridKind kind) : cfg(n, tol, kind) {}
};

int fr_config_create(std::size_t n, double tol, int kind, fr_config** out) {
  return guard([&] { *out = new fr_config(n, tol, kind_of(kind)); });
}

void fr_config_destroy(fr_config* c) { delete c; }

int fr_config_grid(const fr_config* c, double* theta, double* x, double* w) {
  return guard([&] {
    put(c->cfg.grid().theta, theta);
    put(c->cfg.grid().x, x);
    put(c->cfg.grid().weights, w);
  });
}

// dlt (direction 0) / idlt (1) over `cols` columns (column j at in + j*ld),
// spread over `threads` std::threads sharing the immutable config
// (transforms.hpp:15-18 documents that sharing as safe).
int fr_batch(const fr_config* c, int direction, std::size_t cols, std::size_t ld,
             const double* in, double* out, int threads) {
  const std::size_t n = c->cfg.size();
  std::atomic<std::size_t> next{0};
  std::atomic<int> status{0};
  auto worker = [&] {
    for (;;) {
      const std::size_t j = next.fetch_add(1);
      if (j >= cols) break;
      const int rc = guard([&] {
        const std::vector<double> v = vec(in + j * ld, n);
        if (direction == 0)
          put(dlt(legendre_coefficients(v), c->cfg), out + j * ld);
        else
          put(idlt(v, c->cfg).values, out + j * ld);
      });
      if (rc) status = rc;
    }
  };
  if (threads <= 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
  }
  return status;
}

int fr_eval_legendre_direct(std::size_t n, const double* c, std::size_t m, const double* xs,
                            double* out) {
  return guard([&] { put(eval_legendre_direct(legendre_coefficients(vec(c, n)), vec(xs, m)), out); });
}

int fr_eval_chebyshev_direct(std::size_t n, const double* c, std::size_t m, const double* xs,
                             double* out) {
  return guard(
      [&] { put(eval_chebyshev_direct(chebyshev_coefficients(vec(c, n)), vec(xs, m)), out); });
}

int fr_idlt_direct(std::size_t n, const double* f, const double* theta, const double* x,
                   const double* w, double* out) {
  return guard([&] {
    LegendreGrid g{n, vec(theta, n), vec(x, n), vec(w, n)};
    put(idlt_direct(vec(f, n), g).values, out);
  });
}

int fr_cheb_coeffs_of_legendre(std::size_t n, std::size_t m, double* out) {
  return guard([&] { put(cheb_coeffs_of_legendre(n, m), out); });
}

void fr_random_decaying(std::size_t n, double decay, std::uint64_t seed, double* out) {
  put(random_decaying(n, decay, seed), out);
}

std::uint64_t fr_mt19937_64_nth(std::uint64_t seed, std::uint64_t count) {
  std::mt19937_64 r(seed);
  std::uint64_t v = 0;
  for (std::uint64_t i = 0; i < count; ++i) v = r();
  return v;
}

}  // extern "C"
