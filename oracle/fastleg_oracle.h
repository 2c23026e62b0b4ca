/* TEST INFRASTRUCTURE ONLY.
 *
 * C restatement of the reference fastleg hot path (CPU oracle). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker or the timed CPU baseline -- never as
 * the product. Every function cites the reference line it restates
 * (paths relative to /root/reference/proj/include/fastleg/).
 *
 * Pinned against: the compiled reference (oracle/_ref/libfastleg_ref.so,
 * built from the reference headers by oracle/Makefile) and the known-answer
 * values of the reference's own tests (tests/test_oracle_pins.py).
 *
 * Return codes: 0 ok, 1 invalid_argument, 2 domain_error, 3 overflow_error,
 * 4 runtime_error (the reference's exception types).
 */
#ifndef FASTLEG_ORACLE_H
#define FASTLEG_ORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { FO_CHEB1 = 0, FO_CHEBSTAR = 1 };

double fo_reference_angle(size_t n, int kind, size_t k);
int fo_legendre_nodes_weights(size_t n, double* theta, double* x, double* w);
int fo_reference_grid(size_t n, int kind, const double* theta, double* theta_star, double* delta);

int fo_dct_iii(size_t n, int kind, const double* c, double* out);
int fo_dst_iii(size_t n, int kind, const double* c, double* out);
int fo_dct_iii_transpose(size_t n, int kind, const double* g, double* out);
int fo_dst_iii_transpose(size_t n, int kind, const double* g, double* out);

double fo_taylor_term_bound(int kind, int num_terms);
int fo_min_taylor_terms(int kind, double tolerance, int* terms);
int fo_ndct_apply(size_t n, int kind, int num_terms, const double* delta, const double* c,
                  double* f);
int fo_ndct_apply_transpose(size_t n, int kind, int num_terms, const double* delta,
                            const double* g, double* out);
double fo_ndct_error_bound(size_t n, int kind, int num_terms, const double* delta,
                           const double* c);

void fo_lambda_table(size_t max_index, double* table);
int fo_lambda_ratio(double z, const double* table, size_t max_index, double* out);
double fo_leg2cheb_entry(size_t k, size_t n, const double* table, size_t max_index);
int fo_leg2cheb_apply(size_t n, const double* table, size_t max_index, const double* c,
                      double* out);
int fo_leg2cheb_apply_transpose(size_t n, const double* table, size_t max_index,
                                const double* v, double* out);

/* transforms.hpp:42-64 with the grid injected (SURVEY.md 8c protocol 1) */
int fo_dlt_grid(size_t n, int kind, int num_terms, const double* delta, const double* c,
                double* f);
int fo_idlt_grid(size_t n, int kind, int num_terms, const double* delta, const double* weights,
                 const double* f, double* c);

/* oracle.hpp direct evaluations */
int fo_eval_legendre_direct(size_t n, const double* c, size_t m, const double* xs, double* out);
int fo_eval_chebyshev_direct(size_t n, const double* c, size_t m, const double* xs, double* out);
int fo_idlt_direct(size_t n, const double* f, const double* x, const double* w, double* out);
int fo_cheb_coeffs_of_legendre(size_t n, size_t m, double* out);

/* random.hpp input generators (mt19937_64 + Box-Muller) */
void fo_random_decaying(size_t n, double decay, uint64_t seed, double* out);
void fo_uniform_pm1(size_t n, uint64_t seed, double* out);
uint64_t fo_mt19937_64_nth(uint64_t seed, uint64_t count);

#ifdef __cplusplus
}
#endif
#endif
