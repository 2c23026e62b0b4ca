// Bridge from the drop-in headers to the C ABI of libfastleg_b200: status ->
// the reference's exception types, and the batched,
// device-pointer extension for callers that keep data on the GPU.
#pragma once

#include <stdexcept>
#include <string>

#include "fastleg_b200.h"

namespace fastleg {
namespace b200 {

/// Rethrows a failed C-ABI call as the exception the reference throws.
inline void check(fl_status status) {
  switch (status) {
    case FL_OK: return;
    case FL_INVALID_ARGUMENT: throw std::invalid_argument(fl_last_error());
    case FL_DOMAIN_ERROR: throw std::domain_error(fl_last_error());
    case FL_OVERFLOW_ERROR: throw std::overflow_error(fl_last_error());
    default: throw std::runtime_error(fl_last_error());
  }
}

}  // namespace b200
}  // namespace fastleg
