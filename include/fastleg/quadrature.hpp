// Drop-in for proj/include/fastleg/quadrature.hpp. Nodes and weights come
// from the one-thread-per-node asymptotic kernel (fl_nodes_weights); the
// reference grid from fl_reference_grid (same expression order as
// quadrature.hpp:32-36, so theta_star is bit-identical).
#pragma once

#include <cstddef>
#include <vector>

#include "fastleg/b200.hpp"
#include "fastleg/types.hpp"

namespace fastleg {

struct LegendreGrid {
  std::size_t size = 0;
  std::vector<double> theta;    // strictly increasing in (0, pi)
  std::vector<double> x;        // cos(theta), strictly decreasing
  std::vector<double> weights;  // 2 / (dP_N/dtheta)^2
};

struct ReferenceGrid {
  std::size_t size = 0;
  GridKind kind = GridKind::chebstar;
  std::vector<double> theta_star;
  std::vector<double> delta_theta;  // theta - theta_star
};

inline double reference_angle(std::size_t n, GridKind kind, std::size_t k) {
  if (kind == GridKind::cheb1)
    return (static_cast<double>(k) + 0.5) * detail::pi / static_cast<double>(n);
  return (static_cast<double>(k) + 0.75) * detail::pi / (static_cast<double>(n) + 0.5);
}

inline LegendreGrid legendre_nodes_weights(std::size_t n) {
  LegendreGrid g;
  g.size = n;
  g.theta.resize(n);
  g.x.resize(n);
  g.weights.resize(n);
  b200::check(fl_nodes_weights(n, g.theta.data(), g.x.data(), g.weights.data(), nullptr));
  return g;
}

inline ReferenceGrid reference_grid(const LegendreGrid& grid, GridKind kind) {
  ReferenceGrid r;
  r.size = grid.size;
  r.kind = kind;
  r.theta_star.resize(grid.size);
  r.delta_theta.resize(grid.size);
  b200::check(fl_reference_grid(grid.size, static_cast<int>(kind), grid.theta.data(),
                                r.theta_star.data(), r.delta_theta.data(), nullptr));
  return r;
}

}  // namespace fastleg
