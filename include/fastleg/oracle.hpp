// Drop-in for proj/include/fastleg/oracle.hpp: the direct O(N^2) reference
// evaluations, run as device kernels (plain three-term recurrences, sharing
// no code with the FFT-based path, so agreement stays meaningful).
#pragma once

#include <cstddef>
#include <stdexcept>
#include <vector>

#include "fastleg/b200.hpp"
#include "fastleg/quadrature.hpp"
#include "fastleg/types.hpp"

namespace fastleg {

/// sum_n c_n P_n(x_j) for each x_j (domain_error if some |x_j| > 1).
inline std::vector<double> eval_legendre_direct(const CoefficientVector& c,
                                                const std::vector<double>& xs) {
  if (c.basis != Basis::legendre)
    throw std::invalid_argument("eval_legendre_direct: expected Legendre coefficients");
  std::vector<double> out(xs.size());
  b200::check(fl_eval_legendre_direct(c.values.data(), c.values.size(), xs.data(), xs.size(),
                                      out.data(), nullptr));
  return out;
}

/// sum_n c_n T_n(x_j) for each x_j.
inline std::vector<double> eval_chebyshev_direct(const CoefficientVector& c,
                                                 const std::vector<double>& xs) {
  if (c.basis != Basis::chebyshev)
    throw std::invalid_argument("eval_chebyshev_direct: expected Chebyshev coefficients");
  std::vector<double> out(xs.size());
  b200::check(fl_eval_chebyshev_direct(c.values.data(), c.values.size(), xs.data(), xs.size(),
                                       out.data(), nullptr));
  return out;
}

/// c_n = (n + 1/2) sum_k w_k f_k P_n(x_k).
inline CoefficientVector idlt_direct(const std::vector<double>& f, const LegendreGrid& grid) {
  if (f.size() != grid.size) throw std::invalid_argument("idlt_direct: value/grid size mismatch");
  std::vector<double> c(grid.size);
  b200::check(fl_idlt_direct(f.data(), grid.size, grid.x.data(), grid.weights.data(), c.data(),
                             nullptr));
  return legendre_coefficients(std::move(c));
}

/// The n+1 Chebyshev coefficients of P_n from m > n first-kind samples.
inline std::vector<double> cheb_coeffs_of_legendre(std::size_t n, std::size_t m) {
  std::vector<double> out(n + 1);
  b200::check(fl_cheb_coeffs_of_legendre(n, m, out.data(), nullptr));
  return out;
}

}  // namespace fastleg
