// Drop-in for proj/include/fastleg/transforms.hpp: TransformConfig, dlt, idlt.
// TransformConfig owns an immutable device plan (fl_plan: grid, NDCT tables,
// Lambda table) shared by copies of the config, plus host mirrors of the
// grid / TaylorPlan / LambdaCache returned by its accessors.
#pragma once

#include <cstddef>
#include <memory>
#include <stdexcept>
#include <vector>

#include "fastleg/b200.hpp"
#include "fastleg/conversion.hpp"
#include "fastleg/ndct.hpp"
#include "fastleg/quadrature.hpp"
#include "fastleg/types.hpp"

namespace fastleg {

class TransformConfig {
 public:
  explicit TransformConfig(std::size_t n, double tolerance = default_tolerance,
                           GridKind kind = GridKind::chebstar)
      : handle_(create(n, tolerance, kind)),
        grid_(fetch_grid()),
        plan_(fetch_plan()),
        lambda_(n - 1) {}

  std::size_t size() const { return grid_.size; }
  GridKind kind() const { return plan_.kind; }
  double tolerance() const { return plan_.tolerance; }
  const LegendreGrid& grid() const { return grid_; }
  const TaylorPlan& plan() const { return plan_; }
  const LambdaCache& lambda() const { return lambda_; }

  /// The device plan (batched / device-pointer extension, fastleg::b200).
  const fl_plan* handle() const { return handle_.get(); }

 private:
  static std::shared_ptr<fl_plan> create(std::size_t n, double tolerance, GridKind kind) {
    fl_plan* p = nullptr;
    b200::check(fl_plan_create(n, tolerance, static_cast<int>(kind), &p));
    return std::shared_ptr<fl_plan>(p, [](fl_plan* q) { fl_plan_destroy(q); });
  }
  LegendreGrid fetch_grid() const {
    LegendreGrid g;
    g.size = fl_plan_size(handle_.get());
    g.theta.resize(g.size);
    g.x.resize(g.size);
    g.weights.resize(g.size);
    b200::check(fl_plan_grid(handle_.get(), g.theta.data(), g.x.data(), g.weights.data()));
    return g;
  }
  TaylorPlan fetch_plan() const {
    TaylorPlan p;
    p.size = grid_.size;
    p.kind = static_cast<GridKind>(fl_plan_kind(handle_.get()));
    p.tolerance = fl_plan_tolerance(handle_.get());
    p.num_terms = fl_plan_num_terms(handle_.get());
    p.reference.size = p.size;
    p.reference.kind = p.kind;
    p.reference.theta_star.resize(p.size);
    p.reference.delta_theta.resize(p.size);
    b200::check(fl_plan_reference(handle_.get(), p.reference.theta_star.data(),
                                  p.reference.delta_theta.data()));
    return p;
  }

  std::shared_ptr<fl_plan> handle_;
  LegendreGrid grid_;
  TaylorPlan plan_;
  LambdaCache lambda_;
};

/// f_k = sum_n c_n P_n(x_k) at the config's Legendre nodes.
inline std::vector<double> dlt(const CoefficientVector& c, const TransformConfig& config) {
  if (c.basis != Basis::legendre) throw std::invalid_argument("dlt: expected Legendre coefficients");
  if (c.values.size() != config.size())
    throw std::invalid_argument("dlt: coefficient size does not match config");
  std::vector<double> f(c.values.size());
  b200::check(fl_dlt(config.handle(), c.values.data(), f.data(), 1, f.size(), nullptr));
  return f;
}

/// c = D_s M^T T^T D_w f: Legendre coefficients from values at the nodes.
inline CoefficientVector idlt(const std::vector<double>& f, const TransformConfig& config) {
  if (f.size() != config.size()) throw std::invalid_argument("idlt: value size does not match config");
  std::vector<double> c(f.size());
  b200::check(fl_idlt(config.handle(), f.data(), c.data(), 1, c.size(), nullptr));
  return legendre_coefficients(std::move(c));
}

namespace b200 {

/// Batched extension: `batch` columns of config.size() values, column j at
/// ptr + j*ld; pointers may be host or device; `stream` is a cudaStream_t.
inline void dlt_batched(const TransformConfig& config, const double* in, double* out,
                        std::size_t batch, std::size_t ld, void* stream = nullptr) {
  check(fl_dlt(config.handle(), in, out, batch, ld, stream));
}

inline void idlt_batched(const TransformConfig& config, const double* in, double* out,
                         std::size_t batch, std::size_t ld, void* stream = nullptr) {
  check(fl_idlt(config.handle(), in, out, batch, ld, stream));
}

}  // namespace b200

}  // namespace fastleg
