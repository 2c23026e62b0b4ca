/* TEST INFRASTRUCTURE ONLY -- part of the CPU oracle, never the product.
 *
 * FFTW-compatible real-to-real transforms (the four kinds the reference
 * calls: /root/reference/proj/include/fastleg/trig.hpp:63,70,85,91,105,112,
 * 125,132). FFTW3 is absent from this image and from the GPU box, so the
 * compiled reference (oracle/_ref) and the C restatement (fastleg_oracle.c)
 * both sit on this backend. Definitions (unnormalised, FFTW's):
 *   REDFT01: Y_k = X_0 + 2 sum_{j>=1} X_j cos(pi j (k+1/2)/n)
 *   REDFT10: Y_k = 2 sum_j X_j cos(pi (j+1/2) k / n)
 *   RODFT01: Y_k = (-1)^k X_{n-1} + 2 sum_{j<n-1} X_j sin(pi (j+1)(k+1/2)/n)
 *   RODFT10: Y_k = 2 sum_j X_j sin(pi (j+1/2)(k+1)/n)
 * Each is one chirp-z (Bluestein) transform over power-of-two complex FFTs,
 * with per-(kind,n) tables cached under a mutex; execution is reentrant.
 */
#ifndef FASTLEG_ORACLE_R2R_H
#define FASTLEG_ORACLE_R2R_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { R2R_REDFT01 = 4, R2R_REDFT10 = 5, R2R_RODFT01 = 8, R2R_RODFT10 = 9 };

/* returns 0 on success, -1 on a bad kind / n == 0 / allocation failure */
int r2r_execute(int kind, size_t n, const double* in, double* out);

#ifdef __cplusplus
}
#endif
#endif
