/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot path (arxiv 2412.15840, C++ library
 * `ndsylv` under /root/reference/proj). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may call this; the product path
 * (paper_2412_15840_b200/) never links or calls it.
 *
 * Parity pinning: every function here is checked bit-for-bit against the reference
 * library itself, compiled from its own sources into oracle/_ref/ (see Makefile and
 * tests/test_oracle_pins.py), and against the committed golden fixtures under
 * tests/golden/ (made by tests/golden/make_golden.py from oracle/_ref).
 *
 * Layout conventions are the reference's: column-major tensors of complex128
 * (interleaved re,im — std::complex<double> layout, types.hpp:12, tensor.hpp:23-39),
 * square matrices column-major (matrix.hpp:11-30), modes 1-based in the API.
 */
#ifndef NDSYLV_ORACLE_H
#define NDSYLV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_ERR_OTHER = 1,
  ORC_ERR_SINGULAR = 2,
  ORC_ERR_INVALID = 5,
  ORC_ERR_OVERFLOW = 7,
  ORC_ERR_NONFINITE = 9,
};

typedef struct {
  int64_t entries;
  int64_t multiplies;
  double min_abs_denominator;
} orc_backsub_stats;

typedef struct {
  double min_abs_denominator;
  int used_normal_fast_path;
  int64_t flop_estimate;
  int64_t schur_flop_estimate;
  int64_t backsub_entries;
  int64_t backsub_multiplies;
  double transform_seconds;
  double backsub_seconds;
  double inverse_seconds;
} orc_report;

/* tensor.cpp:8-16 — product of dims with overflow check; -1 on invalid, -2 on overflow. */
int64_t orc_checked_total(int n_modes, const int64_t* dims);

/* kernels.cpp:24-44 (mode_product_impl<false>): r = m x_mode x, m square n_mode x n_mode. */
int orc_mode_product(int n_modes, const int64_t* dims, const double* m, int mode, const double* x, double* r);

/* sylvester.cpp:55-61: c = U_N^H x_N ( ... U_1^H x_1 b ). */
int orc_forward_transform(int n_modes, const int64_t* dims, const double* const* u, const double* b, double* c);

/* sylvester.cpp:63-69: x = U_N x_N ( ... U_1 x_1 y ). */
int orc_inverse_transform(int n_modes, const int64_t* dims, const double* const* u, const double* y, double* x);

/* sylvester.cpp:44-53: r = sum_j A_j x_j x. */
int orc_apply_operator(int n_modes, const int64_t* dims, const double* const* a, const double* x, double* r);

/* sylvester.cpp:71-108: in-place triangular solve in descending flat order.
 * On ORC_ERR_SINGULAR, bad_index (length n_modes, 1-based) and bad_den[2] are set. */
int orc_back_substitute(int n_modes, const int64_t* dims, const double* const* t, double* c, double singular_tol,
                        orc_backsub_stats* stats, int64_t* bad_index, double* bad_den);

/* sylvester.cpp:29-33 */
double orc_default_singular_tol(int n_modes, const int64_t* dims, const double* const* t);

/* sylvester.cpp:35-40 */
int orc_numerically_diagonal(int n, const double* t);

/* sylvester.cpp:167-227 minus the Schur step: the whole path given the factors U_j, T_j.
 * flags bit0 = allow_fast_path, bit1 = real_output. x may alias b. */
int orc_solve_schur(int n_modes, const int64_t* dims, const double* const* u, const double* const* t, const double* b,
                    double* x, double singular_tol, unsigned flags, orc_report* rep, int64_t* bad_index,
                    double* bad_den);

/* sylvester.cpp:229-257 */
int64_t orc_flop_estimate(int n_modes, const int64_t* dims);
int64_t orc_schur_flop_estimate(int n_modes, const int64_t* dims);

/* schur.cpp:203-228 (+ pade_exp :230-255, matrix.cpp:48-58 product, :105-113 norm_inf,
 * :143-201 PartialPivLU) — exp(t T) for an upper triangular n x n T. ORC_ERR_INVALID when T has
 * a nonzero strict lower part, ORC_ERR_OTHER when the Pade LU hits a tiny pivot. */
int orc_triangular_exp(int n, const double* t_mat, double t, double* f);

/* ode.cpp:32-87 — OdePropagator(system).at(time) given the Schur factors the constructor would
 * compute (A_j = U_j T_j U_j^H): G = exp(t T_N) x_N ... exp(t T_1) x_1 (sum_j T_j x_j Y0 + C) - C,
 * back_substitute, inverse_transform; flags bit 2 = real_output. Singular as orc_solve_schur. */
int orc_ode_at_schur(int n_modes, const int64_t* dims, const double* const* u, const double* const* t,
                     const double* forcing, const double* initial, double time, double singular_tol, unsigned flags,
                     double* x, int64_t* bad_index, double* bad_den);

/* ode.cpp:93-129 — classical RK4, last step shortened; ORC_ERR_INVALID on a bad step size or
 * step budget, ORC_ERR_NONFINITE when the state leaves finite range. */
int orc_rk4(int n_modes, const int64_t* dims, const double* const* a, const double* forcing, const double* initial,
            double time, double dt, int64_t max_steps, double* x);

/* rng.hpp:12-49 — xoshiro256++ seeded through splitmix64; uniforms from the top 53 bits. */
void orc_xoshiro_uniform(uint64_t seed, int64_t count, double* out);

#ifdef __cplusplus
}
#endif

#endif
