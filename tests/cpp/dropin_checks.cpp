// Drop-in checks of the C++ headers (include/fastleg/*.hpp) over the GPU
// library: the reference's error types and messages, mutable TaylorPlan
// semantics, and the batched extension against single-vector calls.
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "fastleg/fastleg.hpp"

using namespace fastleg;

static int failures = 0;
#define CHECK(cond)                                              \
  do {                                                           \
    if (!(cond)) {                                               \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                \
    }                                                            \
  } while (0)

template <class E, class F>
static bool throws(F&& f, const char* needle = nullptr) {
  try {
    f();
  } catch (const E& e) {
    return needle == nullptr || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  // quadrature.hpp:77, ndct.hpp:49-58, trig.hpp:50, transforms.hpp:43-46
  CHECK(throws<std::invalid_argument>([] { legendre_nodes_weights(0); }, "size must be positive"));
  CHECK(throws<std::domain_error>([] { min_taylor_terms(GridKind::cheb1, 1e-36); }));
  CHECK(throws<std::invalid_argument>([] { min_taylor_terms(GridKind::cheb1, 1.0); }));
  CHECK(throws<std::invalid_argument>([] { dct_iii({}, GridKind::cheb1); }, "dct_iii: empty input"));
  const TransformConfig cfg(64);
  CHECK(cfg.plan().num_terms == 9 && cfg.size() == 64 && cfg.kind() == GridKind::chebstar);
  CHECK(throws<std::invalid_argument>(
      [&] { dlt(chebyshev_coefficients(std::vector<double>(64)), cfg); }, "expected Legendre"));
  CHECK(throws<std::invalid_argument>(
      [&] { dlt(legendre_coefficients(std::vector<double>(63)), cfg); }, "size does not match"));
  std::vector<double> bad(64, 0.0);
  bad[5] = std::numeric_limits<double>::quiet_NaN();
  CHECK(throws<std::invalid_argument>([&] { dlt(legendre_coefficients(bad), cfg); }, "non-finite"));
  CHECK(throws<std::invalid_argument>([&] { ndct_apply(cfg.plan(), bad); }, "ndct_apply: non-finite"));
  CHECK(throws<std::domain_error>(
      [] { eval_legendre_direct(legendre_coefficients({1.0}), {2.0}); }));

  // zero perturbation degenerates to the plain transform, bit for bit (test_ndct.cpp:112-125)
  {
    TaylorPlan plan = plan_ndct(1024, GridKind::cheb1, default_tolerance);
    std::fill(plan.reference.delta_theta.begin(), plan.reference.delta_theta.end(), 0.0);
    const std::vector<double> c = random_decaying(1024, 0.5, 99);
    CHECK(ndct_apply(plan, c) == dct_iii(c, GridKind::cheb1));
    plan.num_terms = 1;
    CHECK(ndct_apply_transpose(plan, c) == dct_iii_transpose(c, GridKind::cheb1));
  }

  // batched extension == single-vector calls
  {
    const std::size_t n = 1024, b = 5;
    const TransformConfig c2(n);
    std::vector<double> in(n * b), out(n * b);
    for (std::size_t j = 0; j < b; ++j) {
      const std::vector<double> v = random_decaying(n, 1.0, 10 + j);
      std::copy(v.begin(), v.end(), in.begin() + j * n);
    }
    b200::dlt_batched(c2, in.data(), out.data(), b, n);
    for (std::size_t j = 0; j < b; ++j) {
      const std::vector<double> v(in.begin() + j * n, in.begin() + (j + 1) * n);
      const std::vector<double> f = dlt(legendre_coefficients(v), c2);
      CHECK(std::equal(f.begin(), f.end(), out.begin() + j * n));
    }
  }

  // vector files round-trip bit-exactly (test_vector_io.cpp:59-72)
  {
    const std::vector<double> v = random_decaying(100, 0.0, 7);
    write_vector("dropin_vec.bin", v, VectorFormat::raw_binary);
    CHECK(read_vector("dropin_vec.bin", VectorFormat::raw_binary) == v);
    write_vector("dropin_vec.csv", v, VectorFormat::csv);
    CHECK(read_vector("dropin_vec.csv", VectorFormat::csv) == v);
    std::remove("dropin_vec.bin");
    std::remove("dropin_vec.csv");
    CHECK(throws<IoError>([] { read_vector("/nonexistent/x", VectorFormat::csv); }));
  }

  std::printf("%s (%d failure(s))\n", failures ? "dropin checks FAILED" : "dropin checks passed",
              failures);
  return failures;
}
