/* TEST INFRASTRUCTURE ONLY -- minimal FFTW3-API shim so the reference headers
 * (/root/reference/proj/include/fastleg/trig.hpp:3,40-46) compile in this
 * image, where FFTW3 is not installed. Only the r2r entry points the
 * reference calls exist; they run oracle/r2r.c. Never shipped. */
#ifndef FASTLEG_ORACLE_FFTW3_SHIM_H
#define FASTLEG_ORACLE_FFTW3_SHIM_H
#include "../r2r.h"

typedef enum {
  FFTW_REDFT01 = R2R_REDFT01,
  FFTW_REDFT10 = R2R_REDFT10,
  FFTW_RODFT01 = R2R_RODFT01,
  FFTW_RODFT10 = R2R_RODFT10
} fftw_r2r_kind;

#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

struct fastleg_shim_plan {
  int n;
  fftw_r2r_kind kind;
};
typedef struct fastleg_shim_plan* fftw_plan;

static inline fftw_plan fftw_plan_r2r_1d(int n, double* in, double* out, fftw_r2r_kind kind,
                                         unsigned flags) {
  (void)in; (void)out; (void)flags;
  if (n <= 0) return 0;
  fftw_plan p = new fastleg_shim_plan;
  p->n = n;
  p->kind = kind;
  return p;
}

static inline void fftw_execute_r2r(const fftw_plan p, double* in, double* out) {
  r2r_execute((int)p->kind, (size_t)p->n, in, out);
}

static inline void fftw_destroy_plan(fftw_plan p) { delete p; }
#endif
