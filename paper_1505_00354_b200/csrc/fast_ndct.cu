#include "common.cuh"
#include "fast_ndct.cuh"
#include "launch.cuh"

namespace flb {

struct FastNdct {
  size_t n;
};

FastNdct* fast_ndct_create(size_t, double, int, const double*) { return nullptr; }
bool fast_ndct_literal_ok(size_t, int) { return false; }
FastNdct* fast_ndct_create_literal(size_t, int, int, const double*, cudaStream_t) { return nullptr; }
void fast_ndct_destroy(FastNdct* p) { delete p; }
void fast_ndct_run(const FastNdct&, int, const double*, size_t, double*, size_t, size_t,
                   const double*, int*, cudaStream_t) {
  fail(FL_RUNTIME_ERROR, "fast ndct: not available");
}

}  // namespace flb
