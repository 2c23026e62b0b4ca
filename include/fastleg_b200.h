/*
 * libfastleg_b200 -- C ABI of the B200-native fast discrete Legendre
 * transform (DLT/IDLT) hot path.
 *
 * This is the drop-in boundary. The reference (`fastleg`, a header-only C++20
 * library) has no C ABI; every entry point below replaces one function of its
 * header API (paths relative to /root/reference/proj/include/fastleg/). The
 * C++ drop-in headers in include/fastleg/*.hpp re-expose these with the
 * reference's exact signatures and exception types.
 *
 * Conventions
 *  - Plain pointers and sizes only. Every double* may point to HOST memory
 *    (the drop-in path: the library stages it through device memory) or to
 *    DEVICE memory (the throughput path: no copies). Pointers of one call
 *    must be all-host or all-device per argument; the library inspects each.
 *  - Batched extension (absent in the reference): `batch`
 *    independent columns, column j at ptr + j*ld (ld >= n). batch = 1,
 *    ld = n is the reference's single-vector call.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 *    synchronous with respect to the host: they return after the results are
 *    complete, as the reference's functions do, so validation errors found on
 *    the device (non-finite input) can be reported as a status.
 *  - Thread-safe: immutable per-size tables are built once under a lock;
 *    scratch is stream-ordered per call (transforms.hpp:15-18, trig.hpp:28-30).
 *  - fp64 throughout. There is no CPU fallback: without a usable CUDA device
 *    every compute entry point returns FL_CUDA_ERROR.
 */
#ifndef FASTLEG_B200_H
#define FASTLEG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the drop-in headers rethrow the reference's exception type
 * (SURVEY.md section 5): */
typedef enum {
  FL_OK = 0,
  FL_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  FL_DOMAIN_ERROR = 2,     /* std::domain_error */
  FL_OVERFLOW_ERROR = 3,   /* std::overflow_error */
  FL_RUNTIME_ERROR = 4,    /* std::runtime_error */
  FL_CUDA_ERROR = 5        /* std::runtime_error (no reference analogue) */
} fl_status;

/* types.hpp:14 GridKind */
typedef enum { FL_CHEB1 = 0, FL_CHEBSTAR = 1 } fl_grid_kind;

/* trig.hpp:55,76,100,118 */
typedef enum { FL_DCT_III = 0, FL_DST_III = 1, FL_DCT_III_T = 2, FL_DST_III_T = 3 } fl_trig_op;

/* Message of the last failing call on this thread (the reference's what()). */
const char* fl_last_error(void);

/* 1 when a CUDA device is usable, else 0 (message in fl_last_error). */
int fl_device_available(void);

/* quadrature.hpp:76-143 legendre_nodes_weights(n): theta ascending in (0,pi),
 * x = cos(theta) descending, weights 2/(dP_N/dtheta)^2; lower half computed,
 * upper half by exact reflection, odd-N middle node (pi/2, 0).
 * n == 0 -> FL_INVALID_ARGUMENT ("legendre_nodes_weights: size must be positive"). */
fl_status fl_nodes_weights(size_t n, double* theta, double* x, double* weights, void* stream);

/* quadrature.hpp:147-158 reference_grid(grid, kind): theta_star and
 * delta_theta = theta - theta_star. */
fl_status fl_reference_grid(size_t n, int kind, const double* theta, double* theta_star,
                            double* delta_theta, void* stream);

/* conversion.hpp:25-30 LambdaCache(max_index): Lambda(z) = Gamma(z+1/2)/Gamma(z+1)
 * for z = 0..max_index (max_index + 1 doubles). */
fl_status fl_lambda_table(size_t max_index, double* table, void* stream);

/* trig.hpp:55-136 dct_iii / dst_iii / dct_iii_transpose / dst_iii_transpose.
 * n == 0 -> FL_INVALID_ARGUMENT ("<op>: empty input"). */
fl_status fl_trig(int op, int kind, size_t n, const double* in, double* out, size_t batch,
                  size_t ld, void* stream);

/* ndct.hpp:98-117 ndct_apply (transpose = 0) and ndct.hpp:121-143
 * ndct_apply_transpose (transpose = 1) for a TaylorPlan given by its fields
 * (kind, size n, num_terms, reference.delta_theta). Validation as
 * ndct.hpp:79-91: non-finite input -> FL_INVALID_ARGUMENT, n^(L-1) overflow
 * guard -> FL_OVERFLOW_ERROR. */
fl_status fl_ndct(int transpose, int kind, size_t n, int num_terms, const double* delta_theta,
                  const double* in, double* out, size_t batch, size_t ld, void* stream);

/* ndct.hpp:147-155 ndct_error_bound(plan, coeffs): min((N max|delta|)^L / L!,
 * C(L)) * ||c||_1, with the two O(N) reductions done on the device, each over
 * its own vector (delta_len = plan.reference.delta_theta.size(), coeffs_len =
 * coeffs.size(); N = n = plan.size). */
fl_status fl_ndct_error_bound(size_t n, int kind, int num_terms, const double* delta_theta,
                              size_t delta_len, const double* coeffs, size_t coeffs_len,
                              double* bound, void* stream);

/* conversion.hpp:100-113 leg2cheb_apply (transpose = 0) and :121-135
 * leg2cheb_apply_transpose (transpose = 1) with the Lambda table of a
 * LambdaCache (lambda_len = max_index + 1 entries, host or device).
 * lambda_len < n -> FL_INVALID_ARGUMENT. */
fl_status fl_leg2cheb(int transpose, size_t n, const double* lambda_table, size_t lambda_len,
                      const double* in, double* out, size_t batch, size_t ld, void* stream);

/* transforms.hpp:19-38 TransformConfig(n, tolerance, kind): an immutable
 * device-resident plan (grid, NDCT plan, Lambda table). Building it is O(N)
 * on the device. */
typedef struct fl_plan fl_plan;
fl_status fl_plan_create(size_t n, double tolerance, int kind, fl_plan** plan);
/* As fl_plan_create but with a caller-supplied grid (theta, x, weights; host
 * or device), i.e. plan_ndct(const LegendreGrid&, ...) at ndct.hpp:61. */
fl_status fl_plan_create_from_grid(size_t n, double tolerance, int kind, const double* theta,
                                   const double* x, const double* weights, fl_plan** plan);
fl_status fl_plan_destroy(fl_plan* plan);
/* Accessors (transforms.hpp:26-31); outputs may be host or device. */
size_t fl_plan_size(const fl_plan* plan);
int fl_plan_kind(const fl_plan* plan);
double fl_plan_tolerance(const fl_plan* plan);
int fl_plan_num_terms(const fl_plan* plan);
fl_status fl_plan_grid(const fl_plan* plan, double* theta, double* x, double* weights);
fl_status fl_plan_reference(const fl_plan* plan, double* theta_star, double* delta_theta);
fl_status fl_plan_lambda(const fl_plan* plan, double* table /* n entries */);

/* transforms.hpp:42-49 dlt: f = NDCT(M c) at the plan's Legendre nodes. */
fl_status fl_dlt(const fl_plan* plan, const double* in, double* out, size_t batch, size_t ld,
                 void* stream);
/* transforms.hpp:54-64 idlt: c = D_s M^T T^T D_w f. */
fl_status fl_idlt(const fl_plan* plan, const double* in, double* out, size_t batch, size_t ld,
                  void* stream);

/* NDCT evaluation mode for plans of kind chebstar (the default grid):
 *   0 = FL_NDCT_LITERAL : L chebstar terms over length-(2N+1) transforms,
 *                         exactly the reference's algorithm (ndct.hpp:98-143);
 *   1 = FL_NDCT_FAST    : same nodes, evaluated internally about the cheb1
 *                         grid over power-of-two real DCTs (SURVEY.md 7 H2
 *                         option B), by the Chebyshev (Jacobi-Anger)
 *                         expansion of cos(n delta), sin(n delta) in n/N --
 *                         14 transforms at 2^-52, tail
 *                         2 sum_{m>=M} |J_m(0.83845)| <= tol -- at every
 *                         power-of-two size (fused on chip for N <= 8192,
 *                         one pack -> multi-pass FFT -> unpack per term
 *                         above).
 * Both are within the reference's certified bound of each other
 * (test_ndct.cpp:173-183). Default FL_NDCT_FAST for dlt/idlt of power-of-two
 * sizes. */
enum { FL_NDCT_LITERAL = 0, FL_NDCT_FAST = 1 };
fl_status fl_plan_set_ndct_mode(fl_plan* plan, int mode);
int fl_plan_ndct_mode(const fl_plan* plan);

/* Process-wide mode of the free functions fl_ndct (ndct.hpp:98-143) and
 * fl_trig (trig.hpp:55-136) at power-of-two N >= 512 (default FL_NDCT_FAST):
 *   FL_NDCT_FAST    : fl_ndct evaluates the same nodes about the cheb1 grid by
 *                     the Chebyshev expansion (either kind; the node offsets
 *                     are re-based exactly, delta' = delta + theta*_kind -
 *                     theta0) whenever the literal L-term evaluation is exact
 *                     to fp64 rounding (its bound min((N max|delta|)^L/L!,
 *                     C(L)) <= 2^-52) and delta is not identically zero; the
 *                     chebstar dct_iii / dst_iii / transposes likewise (zero
 *                     offsets, the sine flavour for the DSTs);
 *   FL_NDCT_LITERAL : the plan's own L Taylor terms on its own grid (chirp-z
 *                     length-(2N+1) transforms for chebstar) -- the ablation.
 * The cheb1 DCT/DST passes and every other size are unaffected. */
fl_status fl_set_free_ndct_mode(int mode);
int fl_free_ndct_mode(void);

/* Legendre -> Chebyshev conversion inside dlt/idlt of plans with n >= 2^14
 * and at most 16 columns:
 *   0 = FL_LEG2CHEB_DIRECT : the reference's O(N^2) triangular product;
 *   1 = FL_LEG2CHEB_FAST   : (default) the asymptotic expansion (mode 2) for
 *       power-of-two n >= 2^16, Toeplitz-Hankel (mode 3) otherwise;
 *   3 = FL_LEG2CHEB_TOEPLITZ : Toeplitz-Hankel factorisation, per parity
 *       A = T .* H with H ~ sum_r l_r l_r^T (pivoted Cholesky, residual
 *       <= 1e-17, so |error| <= 1e-17 ||c||_1), applied as K FFT-based
 *       Toeplitz products;
 *   2 = FL_LEG2CHEB_ASYMPTOTIC : Hale-Townsend asymptotic expansion of
 *       P_n(cos t) at the N cheb1 points (power-of-two N in [2^10, 2^26]):
 *       per level 2M DCT-III/DST-III of diagonally scaled inputs with
 *       diagonal output weights, the low degrees by a chunked three-term
 *       recurrence, then one DCT-II (plans of other sizes keep mode 1).
 *       Replaces conversion.hpp:100-140 like mode 1.
 * fl_plan_leg2cheb_rank returns K for a parity (0 when not built);
 * fl_plan_leg2cheb_asy_info the asymptotic method's expansion terms M, its
 * levels, its length-N transforms per column and its recurrence steps / N
 * (building the method's tables on first call). */
enum {
  FL_LEG2CHEB_DIRECT = 0,
  FL_LEG2CHEB_FAST = 1,
  FL_LEG2CHEB_ASYMPTOTIC = 2,
  FL_LEG2CHEB_TOEPLITZ = 3
};
fl_status fl_plan_set_leg2cheb_mode(fl_plan* plan, int mode);
int fl_plan_leg2cheb_rank(const fl_plan* plan, int parity);
fl_status fl_plan_leg2cheb_asy_info(const fl_plan* plan, int* terms, int* levels,
                                    int* transforms, double* recurrence_steps_per_n);

/* Arithmetic of the direct (dense, triangular) conversion product inside
 * dlt/idlt of plans with more than 16 columns:
 *   0 = FL_GEMM_FP64       : fp64 tensor cores (mma.sync f64, DMMA);
 *   1 = FL_GEMM_INT8_SPLIT : exact split-integer product on the tcgen05 int8
 *       tensor cores: each operand row/column scaled by a power of two and
 *       split into 7 signed 8-bit digits, the 28 digit products with
 *       i + j < 7 accumulated exactly in int32 TMEM accumulators and summed
 *       in fp64 (error <= ~2^-55 max|M row| max|c column| per term, the
 *       order of fp64 rounding). For n a multiple of 256 in [512, 16384];
 *       other sizes use FL_GEMM_FP64.
 * Default FL_GEMM_INT8_SPLIT. fl_plan_gemm_mode returns the current mode. */
enum { FL_GEMM_FP64 = 0, FL_GEMM_INT8_SPLIT = 1 };
fl_status fl_plan_set_gemm_mode(fl_plan* plan, int mode);
int fl_plan_gemm_mode(const fl_plan* plan);

/* How dlt / idlt evaluate (transforms.hpp:42-64):
 *   0 = FL_DLT_FACTORED : the reference's factorisation, f = NDCT(M c) and
 *                         c = D_s M^T NDCT^T(D_w f) (conversion + NDCT);
 *   1 = FL_DLT_DIRECT   : the same transform as one dense product per parity,
 *       f = P c and c = D_s P^T D_w f with P_kn = P_n(cos theta_k) evaluated
 *       (double-double, once per plan) at the reference's angles
 *       theta*_kind(k) + delta_k, on the int8 tcgen05 tensor cores with the
 *       split arithmetic of FL_GEMM_INT8_SPLIT (exact digit products, fp64
 *       recombination). The parity split (P_n(-x) = (-1)^n P_n(x)) halves
 *       it: 2 (N/2)^2 MACs per column, N^2/2 -- against the factored path's
 *       N^2/4 conversion plus the ~14-term NDCT, which it beats for
 *       N <= 8192 on B200 (the paper's own direct/fast crossover is
 *       N ~ 5000).
 * FL_DLT_DIRECT (default) applies to n a multiple of 256 in [512, 8192],
 * more than 16 columns and FL_GEMM_INT8_SPLIT; everything else is factored.
 * A non-finite input column raises invalid_argument with the factored
 * path's message (ndct_apply[_transpose]: non-finite input).
 * fl_plan_uses_direct tells which one a call with `batch` columns takes. */
enum { FL_DLT_FACTORED = 0, FL_DLT_DIRECT = 1 };
fl_status fl_plan_set_dlt_method(fl_plan* plan, int method);
int fl_plan_dlt_method(const fl_plan* plan);
int fl_plan_uses_direct(const fl_plan* plan, size_t batch);

/* The plan's conversion step alone, exactly as dlt/idlt run it (same
 * leg2cheb / gemm mode selection): out = M in (transpose = 0, the first step
 * of transforms.hpp:47) or (m + 1/2) M^T in (transpose = 1, the last step of
 * transforms.hpp:62). Host or device pointers, columns of stride ld. */
fl_status fl_plan_leg2cheb(const fl_plan* plan, int transpose, const double* in, double* out,
                           size_t batch, size_t ld, void* stream);

/* The plan's NDCT step alone, as dlt/idlt run it (same FL_NDCT_* mode):
 * out = NDCT(in) (transpose = 0, transforms.hpp:48) or NDCT^T(in) (1, the
 * unweighted ndct_apply_transpose of transforms.hpp:60).
 * fl_plan_ndct_terms: transforms per column it evaluates (fast mode: the
 * Chebyshev / Jacobi-Anger expansion about cheb1, 14 terms at 2^-52, at
 * every power-of-two size; the plan's own L when literal). */
fl_status fl_plan_ndct(const fl_plan* plan, int transpose, const double* in, double* out,
                       size_t batch, size_t ld, void* stream);
int fl_plan_ndct_terms(const fl_plan* plan);

/* Term-parallel pieces of dlt / idlt (multi-GPU extension for one large
 * vector, C5). Both stages of fl_dlt are sums of independent terms, so P
 * ranks each take a slice and one collective sums the partials
 * (paper_1505_00354_b200/distributed.py):
 *   FL_STAGE_LEG2CHEB : the conversion the plan runs for one column, as a
 *                       sum of terms: with the asymptotic expansion (power-of-
 *                       two n >= 2^16, FL_LEG2CHEB_FAST) its (level, m)
 *                       DCT/DST pairs, then its recurrence bands (each partial
 *                       ends with the DCT-II, which is linear); with
 *                       Toeplitz-Hankel chat = sum_{r in [lo,hi)} D(l_r) T
 *                       D(l_r) c, its rank terms (idlt: M^T with (m+1/2));
 *   FL_STAGE_NDCT     : f = sum_{m in [lo,hi)} term m of the fast-mode NDCT
 *                       (the Chebyshev-expansion terms about cheb1, 14 at
 *                       2^-52; idlt: the transpose, with the quadrature
 *                       weights).
 * One column; needs the fast paths (n >= 2^15 and a power of two > 8192).
 * fl_plan_stage_terms gives the number of terms of a stage,
 * fl_plan_stage_cost a term's relative cost (the asymptotic conversion's
 * terms differ: a (level, m) pair is two length-n transforms, a recurrence
 * band its pairs x degrees; all other terms 1) for a balanced split. */
enum { FL_STAGE_LEG2CHEB = 0, FL_STAGE_NDCT = 1 };
fl_status fl_plan_stage_terms(const fl_plan* plan, int stage, int* count);
fl_status fl_plan_stage_cost(const fl_plan* plan, int stage, int term, double* cost);
fl_status fl_dlt_stage(const fl_plan* plan, int inverse, int stage, int lo, int hi,
                       const double* in, double* out, void* stream);

/* Distributed four-step NDCT of one vector over P ranks (C5 sharded, the
 * multi-GPU form north_star names; paper_1505_00354_b200/distributed.py
 * drives it with NCCL). Replaces, for a vector spread over P GPUs, the
 * per-term FFTW calls of ndct_apply / ndct_apply_transpose (ndct.hpp:98-143,
 * trig.hpp:66-73): every term's N/2-point FFT is L1 x L2 (L1 L2 = N/2), the
 * L2-point FFTs on the rank owning a symmetric set of residues m1 (mod L1)
 * of the packed input, the L1-point FFTs on the rank owning a block of k2;
 * ONE all-to-all per group of terms between them (the caller's collective:
 * per peer and term fl_fs_coef_count complex entries). The coefficient side
 * lives in a residue layout (fl_fs_to_residue / fl_fs_from_residue map a
 * natural full vector to the [rank][res_max][2 L2] slabs of a reduce-scatter /
 * all-gather), the value side in natural blocks of N/P (fl_fs_values maps
 * them to / from the uniform [peer][N/P^2] exchange layout of the final
 * all-to-all). Needs a fast-mode plan (power-of-two N), P a power of two,
 * 2P <= L1 and N <= 2^27. All pointers device; stream-ordered on `stream`.
 *   fl_fs_info: n, L, L1, L2, KB = L2/P, B = N/P, residues of this rank,
 *               max residues over ranks, world, rank (10 entries).
 *   fl_fs_ndct_part(transpose, part, t0, t1, in, out, work, first):
 *     forward part 1: in = residue-layout chat, out = coefficient exchange
 *       (send); part 2: in = received exchange, out = value exchange layout
 *       (accumulated over term groups unless first).
 *     transpose part 1: in = value exchange layout (received), out = send;
 *       part 2: in = received, out = residue layout (accumulated unless first).
 *     work: fl_fs_work_elems complex entries for t1 - t0 terms.
 *   fl_fs_check: synchronises `stream`; FL_INVALID_ARGUMENT with the
 *     reference's message when a part-1 call saw a non-finite input. */
typedef struct fl_fs fl_fs;
fl_status fl_fs_create(const fl_plan* plan, int world, int rank, fl_fs** fs);
fl_status fl_fs_destroy(fl_fs* fs);
fl_status fl_fs_info(const fl_fs* fs, size_t* info);
fl_status fl_fs_coef_count(const fl_fs* fs, int transpose, int peer, int send, size_t* count);
size_t fl_fs_work_elems(const fl_fs* fs, int terms);
fl_status fl_fs_to_residue(const fl_fs* fs, const double* full, double* slabs, void* stream);
fl_status fl_fs_from_residue(const fl_fs* fs, const double* slabs, double* full, void* stream);
fl_status fl_fs_values(const fl_fs* fs, int to_block, const double* in, double* out, void* stream);
fl_status fl_fs_ndct_part(const fl_fs* fs, int transpose, int part, int t0, int t1, const void* in,
                          void* out, void* work, int first, void* stream);
fl_status fl_fs_check(const fl_fs* fs, int transpose, void* stream);

/* oracle.hpp:19-153 direct O(N^2) evaluations, on the device (independent of
 * the fast path: plain three-term recurrences, no FFTs).
 *   eval_legendre_direct / eval_chebyshev_direct: out[j] = sum_n c_n P_n(xs[j])
 *     (resp. T_n); any |xs[j]| > 1 -> FL_DOMAIN_ERROR.
 *   idlt_direct: c_m = (m + 1/2) sum_k w_k f_k P_m(x_k).
 *   cheb_coeffs_of_legendre: the n+1 Chebyshev coefficients of P_n from m
 *     first-kind samples; m <= n -> FL_INVALID_ARGUMENT. */
fl_status fl_eval_legendre_direct(const double* c, size_t n, const double* xs, size_t m,
                                  double* out, void* stream);
fl_status fl_eval_chebyshev_direct(const double* c, size_t n, const double* xs, size_t m,
                                   double* out, void* stream);
fl_status fl_idlt_direct(const double* f, size_t n, const double* x, const double* weights,
                         double* out, void* stream);
fl_status fl_cheb_coeffs_of_legendre(size_t n, size_t m, double* out, void* stream);

/* random.hpp:15-55 input generators (host memory; std::mt19937_64 +
 * Box-Muller): random_decaying(n, decay, seed), and the uniform [-1,1)
 * recipe u = 2*((r()>>11)*2^-53) - 1 of SURVEY.md 8d (C4). Batched: column
 * j uses seed + j. `threads` host threads (0 = hardware concurrency). */
void fl_random_decaying(size_t n, double decay, uint64_t seed, double* out, size_t batch,
                        int threads);
void fl_random_uniform_pm1(size_t n, uint64_t seed, double* out, size_t batch, int threads);

/* vector_io.hpp:22-102: the on-disk vector formats
 * either side of the transforms, staged straight to / from device memory.
 * format 0 = csv (one value per line), 1 = raw_binary ("FLEGVEC1", uint64 LE
 * count, binary64 LE values). `out` / `in` may be device or host pointers.
 *   fl_load_vector: the binary payload is read in chunks into two pinned
 *     buffers whose async H2D copies overlap the next chunk's read; csv is
 *     parsed into a pinned buffer and copied once. *count = the vector's
 *     length; capacity < count -> FL_INVALID_ARGUMENT (nothing copied).
 *   fl_save_vector: D2H in chunks into pinned buffers, written as they land.
 * Errors: FL_RUNTIME_ERROR with the reference's IoError messages (cannot
 * open, bad magic, truncated header / payload, not a number). */
fl_status fl_load_vector(const char* path, int format, double* out, size_t capacity,
                         size_t* count, void* stream);
fl_status fl_save_vector(const char* path, int format, const double* in, size_t n, void* stream);

/* Number of kernels this library has launched since load (telemetry for the
 * bench's gpu_launches field). */
uint64_t fl_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FASTLEG_B200_H */
