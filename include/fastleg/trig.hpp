// Drop-in for proj/include/fastleg/trig.hpp: DCT-III / DST-III on either
// grid and their exact transposes, in the reference's normalisation
//   dct_iii(c)_k = sum_n c_n cos(n theta*_k),  dst_iii(c)_k = sum_n c_n sin(n theta*_k)
// computed by the sm_100a engine (fused real-FFT kernels for power-of-two
// cheb1 sizes, chirp-z over power-of-two FFTs otherwise).
#pragma once

#include <vector>

#include "fastleg/b200.hpp"
#include "fastleg/types.hpp"

namespace fastleg {

namespace detail {
inline std::vector<double> trig_call(int op, const std::vector<double>& v, GridKind kind) {
  std::vector<double> out(v.size());
  b200::check(fl_trig(op, static_cast<int>(kind), v.size(), v.data(), out.data(), 1, v.size(),
                      nullptr));
  return out;
}
}  // namespace detail

inline std::vector<double> dct_iii(const std::vector<double>& c, GridKind kind) {
  return detail::trig_call(FL_DCT_III, c, kind);
}

inline std::vector<double> dst_iii(const std::vector<double>& c, GridKind kind) {
  return detail::trig_call(FL_DST_III, c, kind);
}

inline std::vector<double> dct_iii_transpose(const std::vector<double>& g, GridKind kind) {
  return detail::trig_call(FL_DCT_III_T, g, kind);
}

inline std::vector<double> dst_iii_transpose(const std::vector<double>& g, GridKind kind) {
  return detail::trig_call(FL_DST_III_T, g, kind);
}

}  // namespace fastleg
