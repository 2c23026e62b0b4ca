// Drop-in for proj/include/fastleg/ndct.hpp: the Taylor-series NDCT
// (Chebyshev evaluation at the Legendre nodes). TaylorPlan stays a mutable
// host aggregate -- every call passes its current fields to the device
// (tests edit delta_theta / num_terms after planning, test_ndct.cpp:114-153).
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

#include "fastleg/b200.hpp"
#include "fastleg/quadrature.hpp"
#include "fastleg/types.hpp"

namespace fastleg {

struct TaylorPlan {
  std::size_t size = 0;
  GridKind kind = GridKind::chebstar;
  double tolerance = 0.0;
  int num_terms = 0;  // L
  ReferenceGrid reference;
};

/// C(L): 0.83845^L / L! (cheb1) or ((6 pi)^L L!)^-1 (chebstar).
inline double taylor_term_bound(GridKind kind, int num_terms) {
  if (num_terms < 0) throw std::invalid_argument("taylor_term_bound: negative term count");
  const double q = kind == GridKind::cheb1 ? 0.83845 : 1.0 / (6.0 * detail::pi);
  double bound = 1.0;
  for (int l = 1; l <= num_terms; ++l) bound *= q / static_cast<double>(l);
  return bound;
}

inline constexpr int max_taylor_terms = 30;

inline int min_taylor_terms(GridKind kind, double tolerance) {
  if (!(tolerance > 0.0 && tolerance < 1.0))
    throw std::invalid_argument("min_taylor_terms: tolerance must lie in (0, 1)");
  double bound = 1.0;
  const double q = kind == GridKind::cheb1 ? 0.83845 : 1.0 / (6.0 * detail::pi);
  for (int l = 1; l <= max_taylor_terms; ++l) {
    bound *= q / static_cast<double>(l);
    if (bound <= tolerance) return l;
  }
  throw std::domain_error("min_taylor_terms: tolerance unattainable with <= 30 terms");
}

inline TaylorPlan plan_ndct(const LegendreGrid& grid, GridKind kind, double tolerance) {
  TaylorPlan plan;
  plan.size = grid.size;
  plan.kind = kind;
  plan.tolerance = tolerance;
  plan.num_terms = min_taylor_terms(kind, tolerance);
  plan.reference = reference_grid(grid, kind);
  return plan;
}

inline TaylorPlan plan_ndct(std::size_t n, GridKind kind, double tolerance) {
  return plan_ndct(legendre_nodes_weights(n), kind, tolerance);
}

namespace detail {
inline std::vector<double> ndct_call(int transpose, const TaylorPlan& plan,
                                     const std::vector<double>& v, const char* where) {
  if (v.size() != plan.size)
    throw std::invalid_argument(std::string(where) + ": input size does not match plan");
  if (plan.reference.delta_theta.size() != plan.size)
    throw std::invalid_argument(std::string(where) + ": plan perturbations do not match size");
  std::vector<double> out(v.size());
  b200::check(fl_ndct(transpose, static_cast<int>(plan.kind), plan.size, plan.num_terms,
                      plan.reference.delta_theta.data(), v.data(), out.data(), 1, v.size(),
                      nullptr));
  return out;
}
}  // namespace detail

/// f_k ~= sum_n c_n cos(n theta_k) at the plan's Legendre angles.
inline std::vector<double> ndct_apply(const TaylorPlan& plan, const std::vector<double>& coeffs) {
  return detail::ndct_call(0, plan, coeffs, "ndct_apply");
}

/// Exact transpose of ndct_apply.
inline std::vector<double> ndct_apply_transpose(const TaylorPlan& plan,
                                                const std::vector<double>& values) {
  return detail::ndct_call(1, plan, values, "ndct_apply_transpose");
}

/// min((N max|dtheta|)^L / L!, C(L)) * ||c||_1, reductions on the device.
inline double ndct_error_bound(const TaylorPlan& plan, const std::vector<double>& coeffs) {
  double bound = 0.0;
  b200::check(fl_ndct_error_bound(plan.size, static_cast<int>(plan.kind), plan.num_terms,
                                  plan.reference.delta_theta.data(),
                                  plan.reference.delta_theta.size(), coeffs.data(),
                                  coeffs.size(), &bound, nullptr));
  return bound;
}

}  // namespace fastleg
