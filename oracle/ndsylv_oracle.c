/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see ndsylv_oracle.h). Never linked by the product.
 *
 * Scalar C11 restatement of the reference hot path. Arithmetic uses C99 `double _Complex`,
 * which GCC lowers exactly as it lowers std::complex<double> in the reference (inline
 * multiply with the __muldc3 NaN-recovery fallback, __divdc3 for division, cabs for
 * std::abs), and loops keep the reference's summation order, so results are bitwise
 * identical to the reference build in oracle/_ref (pinned by tests/test_oracle_pins.py).
 */
#define _POSIX_C_SOURCE 199309L
#include "ndsylv_oracle.h"

#include <complex.h>
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef double _Complex cxd;

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* tensor.cpp:8-16 */
int64_t orc_checked_total(int n_modes, const int64_t* dims) {
  if (n_modes < 1) return -1;
  int64_t total = 1;
  for (int j = 0; j < n_modes; ++j) {
    if (dims[j] < 1) return -1;
    if (__builtin_mul_overflow(total, dims[j], &total)) return -2;
  }
  return total;
}

/* kernels.cpp:9-21 — the (inner, n, outer) view of mode `mode` (1-based). */
static void slab(int n_modes, const int64_t* dims, int mode, int64_t* inner, int64_t* n, int64_t* outer) {
  *inner = 1;
  *outer = 1;
  *n = dims[mode - 1];
  for (int j = 0; j < mode - 1; ++j) *inner *= dims[j];
  for (int j = mode; j < n_modes; ++j) *outer *= dims[j];
}

/* kernels.cpp:24-44 — serial twin (kernels.cpp:92); same loop nest and summation order. */
int orc_mode_product(int n_modes, const int64_t* dims, const double* m_raw, int mode, const double* x_raw,
                     double* r_raw) {
  if (mode < 1 || mode > n_modes) return ORC_ERR_INVALID;
  int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  int64_t inner, n, outer;
  slab(n_modes, dims, mode, &inner, &n, &outer);
  const cxd* m = (const cxd*)m_raw;
  const cxd* x = (const cxd*)x_raw;
  cxd* r = (cxd*)r_raw;
  memset(r, 0, (size_t)total * sizeof(cxd)); /* NDTensor::zeros, kernels.cpp:28 */
  const int64_t block = inner * n;
  for (int64_t b = 0; b < outer; ++b) {
    for (int64_t i = 0; i < n; ++i) {
      cxd* out = r + b * block + i * inner;
      for (int64_t k = 0; k < n; ++k) {
        const cxd mik = m[i + k * n]; /* Matrix::operator() column-major, matrix.hpp:29-30 */
        const cxd* in = x + b * block + k * inner;
        for (int64_t a = 0; a < inner; ++a) out[a] += mik * in[a];
      }
    }
  }
  return ORC_OK;
}

/* matrix.cpp:34-39 */
static void adjoint(int64_t n, const cxd* u, cxd* uh) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) uh[j + i * n] = conj(u[i + j * n]);
}

/* sylvester.cpp:55-69 — modes applied 1..N, a fresh tensor per mode. */
static int transform(int n_modes, const int64_t* dims, const double* const* u, const double* in, double* out,
                     int use_adjoint) {
  int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  cxd* cur = (cxd*)malloc((size_t)total * sizeof(cxd));
  cxd* nxt = (cxd*)malloc((size_t)total * sizeof(cxd));
  if (!cur || !nxt) {
    free(cur);
    free(nxt);
    return ORC_ERR_OTHER;
  }
  memcpy(cur, in, (size_t)total * sizeof(cxd));
  for (int j = 1; j <= n_modes; ++j) {
    const int64_t n = dims[j - 1];
    const double* m = u[j - 1];
    cxd* tmp = NULL;
    if (use_adjoint) {
      tmp = (cxd*)malloc((size_t)(n * n) * sizeof(cxd));
      adjoint(n, (const cxd*)u[j - 1], tmp);
      m = (const double*)tmp;
    }
    orc_mode_product(n_modes, dims, m, j, (const double*)cur, (double*)nxt);
    free(tmp);
    cxd* s = cur;
    cur = nxt;
    nxt = s;
  }
  memcpy(out, cur, (size_t)total * sizeof(cxd));
  free(cur);
  free(nxt);
  return ORC_OK;
}

int orc_forward_transform(int n_modes, const int64_t* dims, const double* const* u, const double* b, double* c) {
  return transform(n_modes, dims, u, b, c, 1);
}

int orc_inverse_transform(int n_modes, const int64_t* dims, const double* const* u, const double* y, double* x) {
  return transform(n_modes, dims, u, y, x, 0);
}

/* sylvester.cpp:44-53 — r = 0; r += 1.0 * (A_j x_j x) per mode (add_scaled, kernels.cpp:81-88). */
int orc_apply_operator(int n_modes, const int64_t* dims, const double* const* a, const double* x, double* r_raw) {
  int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  cxd* term = (cxd*)malloc((size_t)total * sizeof(cxd));
  if (!term) return ORC_ERR_OTHER;
  cxd* r = (cxd*)r_raw;
  memset(r, 0, (size_t)total * sizeof(cxd));
  for (int j = 1; j <= n_modes; ++j) {
    orc_mode_product(n_modes, dims, a[j - 1], j, x, (double*)term);
    const cxd alpha = 1.0;
    for (int64_t i = 0; i < total; ++i) r[i] += alpha * term[i];
  }
  free(term);
  return ORC_OK;
}

/* matrix.cpp:99-103 */
static double norm_frobenius(int64_t n, const cxd* t) {
  double s = 0.0;
  for (int64_t i = 0; i < n * n; ++i) {
    const double re = creal(t[i]), im = cimag(t[i]);
    s += re * re + im * im; /* std::norm for double: x*x + y*y */
  }
  return sqrt(s);
}

/* sylvester.cpp:29-33 */
double orc_default_singular_tol(int n_modes, const int64_t* dims, const double* const* t) {
  double s = 0.0;
  for (int j = 0; j < n_modes; ++j) s += norm_frobenius(dims[j], (const cxd*)t[j]);
  return DBL_EPSILON * s;
}

/* sylvester.cpp:35-40 */
int orc_numerically_diagonal(int n, const double* t_raw) {
  const cxd* t = (const cxd*)t_raw;
  double off2 = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < j; ++i) {
      const double re = creal(t[i + (int64_t)j * n]), im = cimag(t[i + (int64_t)j * n]);
      off2 += re * re + im * im;
    }
  return sqrt(off2) <= 1e-12 * (1.0 + norm_frobenius(n, t));
}

/* Decode a 0-based flat index into the 1-based multi-index (tensor.cpp:29-41 inverted). */
static void decode(int n_modes, const int64_t* dims, int64_t flat, int64_t* multi) {
  for (int j = 0; j < n_modes; ++j) {
    multi[j] = flat % dims[j] + 1;
    flat /= dims[j];
  }
}

/* sylvester.cpp:71-108. The MultiIndexCursor (tensor.cpp:68-93, paper Alg. 2) visits flat
 * positions total..1 with i_1 fastest; we keep the decoded multi-index in `cur` and step it
 * the same way (odometer decrement). */
int orc_back_substitute(int n_modes, const int64_t* dims, const double* const* t_raw, double* c_raw,
                        double singular_tol, orc_backsub_stats* stats, int64_t* bad_index, double* bad_den) {
  int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  int64_t strides[64];
  int64_t cur[64];
  if (n_modes > 64) return ORC_ERR_INVALID;
  int64_t acc = 1;
  for (int j = 0; j < n_modes; ++j) {
    strides[j] = acc;
    acc *= dims[j];
    cur[j] = dims[j];
  }
  cxd* data = (cxd*)c_raw;
  orc_backsub_stats st = {0, 0, INFINITY};
  for (int64_t index = total; index >= 1; --index) {
    const int64_t flat = index - 1;
    cxd num = data[flat];
    cxd den = 0.0;
    for (int j = 0; j < n_modes; ++j) {
      const cxd* t = (const cxd*)t_raw[j];
      const int64_t ij = cur[j], nj = dims[j];
      den += t[(ij - 1) + (ij - 1) * nj];
      const int64_t stride = strides[j];
      for (int64_t k = ij + 1; k <= nj; ++k) num -= t[(ij - 1) + (k - 1) * nj] * data[flat + (k - ij) * stride];
      st.multiplies += nj - ij;
    }
    const double aden = cabs(den);
    st.min_abs_denominator = fmin(st.min_abs_denominator, aden);
    if (aden <= singular_tol) {
      if (bad_index) memcpy(bad_index, cur, (size_t)n_modes * sizeof(int64_t));
      if (bad_den) {
        bad_den[0] = creal(den);
        bad_den[1] = cimag(den);
      }
      if (stats) *stats = st;
      return ORC_ERR_SINGULAR;
    }
    data[flat] = num / den;
    ++st.entries;
    /* MultiIndexCursor::next, tensor.cpp:77-93 */
    if (cur[0] >= 2) {
      --cur[0];
    } else {
      int k = 1;
      while (k < n_modes && cur[k] == 1) ++k;
      if (k < n_modes) {
        --cur[k];
        for (int j = 0; j < k; ++j) cur[j] = dims[j];
      }
    }
  }
  if (stats) *stats = st;
  return ORC_OK;
}

/* sylvester.cpp:119-141 — eigenvalue sums in cursor order; first offender (descending) wins. */
static int eigenvalue_sums(int n_modes, const int64_t* dims, const double* const* t_raw, double tol, cxd* sums,
                           double* min_abs, int64_t* bad_index, double* bad_den) {
  const int64_t total = orc_checked_total(n_modes, dims);
  double best = INFINITY;
  int64_t multi[64];
  for (int64_t index = total; index >= 1; --index) {
    decode(n_modes, dims, index - 1, multi);
    cxd den = 0.0;
    for (int j = 0; j < n_modes; ++j) {
      const cxd* t = (const cxd*)t_raw[j];
      den += t[(multi[j] - 1) + (multi[j] - 1) * dims[j]];
    }
    const double aden = cabs(den);
    best = fmin(best, aden);
    if (aden <= tol) {
      if (bad_index) memcpy(bad_index, multi, (size_t)n_modes * sizeof(int64_t));
      if (bad_den) {
        bad_den[0] = creal(den);
        bad_den[1] = cimag(den);
      }
      return ORC_ERR_SINGULAR;
    }
    sums[index - 1] = den;
  }
  *min_abs = best;
  return ORC_OK;
}

/* sylvester.cpp:17-27 validation is the caller's (shapes are implied by dims here);
 * sylvester.cpp:167-227 minus the Schur step. */
int orc_solve_schur(int n_modes, const int64_t* dims, const double* const* u, const double* const* t,
                    const double* b, double* x, double singular_tol, unsigned flags, orc_report* rep,
                    int64_t* bad_index, double* bad_den) {
  if (n_modes < 2) return ORC_ERR_INVALID;
  const int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  orc_report r;
  memset(&r, 0, sizeof r);
  r.flop_estimate = orc_flop_estimate(n_modes, dims);
  r.schur_flop_estimate = orc_schur_flop_estimate(n_modes, dims);
  const double tol = singular_tol > 0.0 ? singular_tol : orc_default_singular_tol(n_modes, dims, t);
  int diagonal_route = (flags & 1u) != 0;
  for (int j = 0; diagonal_route && j < n_modes; ++j)
    if (!orc_numerically_diagonal((int)dims[j], t[j])) diagonal_route = 0;
  cxd* c = (cxd*)malloc((size_t)total * sizeof(cxd));
  if (!c) return ORC_ERR_OTHER;
  int rc = ORC_OK;
  if (diagonal_route) {
    cxd* sums = (cxd*)malloc((size_t)total * sizeof(cxd));
    if (!sums) {
      free(c);
      return ORC_ERR_OTHER;
    }
    rc = eigenvalue_sums(n_modes, dims, t, tol, sums, &r.min_abs_denominator, bad_index, bad_den);
    if (rc == ORC_OK) {
      double t0 = now_seconds();
      orc_forward_transform(n_modes, dims, u, b, (double*)c);
      r.transform_seconds = now_seconds() - t0;
      t0 = now_seconds();
      for (int64_t i = 0; i < total; ++i) c[i] /= sums[i];
      r.backsub_seconds = now_seconds() - t0;
      t0 = now_seconds();
      orc_inverse_transform(n_modes, dims, u, (const double*)c, x);
      r.inverse_seconds = now_seconds() - t0;
      r.used_normal_fast_path = 1;
    }
    free(sums);
  } else {
    double t0 = now_seconds();
    orc_forward_transform(n_modes, dims, u, b, (double*)c);
    r.transform_seconds = now_seconds() - t0;
    t0 = now_seconds();
    orc_backsub_stats st;
    rc = orc_back_substitute(n_modes, dims, t, (double*)c, tol, &st, bad_index, bad_den);
    r.backsub_seconds = now_seconds() - t0;
    r.backsub_entries = st.entries;
    r.backsub_multiplies = st.multiplies;
    r.min_abs_denominator = st.min_abs_denominator;
    if (rc == ORC_OK) {
      t0 = now_seconds();
      orc_inverse_transform(n_modes, dims, u, (const double*)c, x);
      r.inverse_seconds = now_seconds() - t0;
    }
  }
  free(c);
  if (rc == ORC_OK && (flags & 2u)) /* real_output, sylvester.cpp:223-224 */
    for (int64_t i = 0; i < total; ++i) x[2 * i + 1] = 0.0;
  if (rep) *rep = r;
  return rc;
}

/* sylvester.cpp:229-241 */
int64_t orc_flop_estimate(int n_modes, const int64_t* dims) {
  const int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return -1;
  int64_t sum = 0, factor = 0, flops = 0;
  for (int j = 0; j < n_modes; ++j)
    if (__builtin_add_overflow(sum, dims[j], &sum)) return -1;
  if (__builtin_mul_overflow(sum, (int64_t)5, &factor) || __builtin_add_overflow(factor, (int64_t)1 - n_modes, &factor))
    return -1;
  if (__builtin_mul_overflow(total, factor, &flops)) return -1;
  return flops;
}

/* sylvester.cpp:243-257 */
int64_t orc_schur_flop_estimate(int n_modes, const int64_t* dims) {
  if (orc_checked_total(n_modes, dims) < 0) return -1;
  int64_t sum_cubes = 0, flops = 0;
  for (int j = 0; j < n_modes; ++j) {
    int64_t sq = 0, cube = 0;
    if (__builtin_mul_overflow(dims[j], dims[j], &sq) || __builtin_mul_overflow(sq, dims[j], &cube) ||
        __builtin_add_overflow(sum_cubes, cube, &sum_cubes))
      return -1;
  }
  if (__builtin_mul_overflow(sum_cubes, (int64_t)25, &flops)) return -1;
  return flops;
}

/* rng.hpp:12-43 */
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void orc_xoshiro_uniform(uint64_t seed, int64_t count, double* out) {
  uint64_t s[4];
  uint64_t sm = seed;
  for (int w = 0; w < 4; ++w) {
    sm += 0x9e3779b97f4a7c15ULL;
    uint64_t z = sm;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    s[w] = z ^ (z >> 31);
  }
  for (int64_t i = 0; i < count; ++i) {
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    out[i] = (double)(result >> 11) * 0x1.0p-53;
  }
}
